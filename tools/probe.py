"""Read-probe variants (profiling): LDG vs cp.async, CTAs per SM."""
import ctypes as C, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2001_05585_b200 as T
from paper_2001_05585_b200 import _capi
lib = _capi.load()
n = 1 << 30
x = T.generate("uniform", 0, n)
st = torch.cuda.current_stream()
sp = C.c_void_p(st.cuda_stream)
xp = C.c_void_p(x.data_ptr())
for mode, ctas in [("ldg", 8), ("ldg", 4), ("ldg", 3), ("async", 8), ("async", 6), ("async", 4), ("async", 3)]:
    os.environ["TCR_PROBE"] = mode
    os.environ["TCR_PROBE_CTAS"] = str(ctas)
    lib.tcr_enable_profiling_knobs()
    ts = []
    for rep in range(5):
        for _ in range(2):
            _capi.check(lib.tcr_read_probe_async(xp, 2 * n, sp))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(10):
            _capi.check(lib.tcr_read_probe_async(xp, 2 * n, sp))
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) / 10)
    ms = statistics.median(ts)
    print(f"{mode:6s} ctas/SM={ctas}: {ms*1e3:.1f} us  {2*n/ms/1e9:.3f} TB/s", flush=True)
