import sys, ctypes as C, statistics
sys.path.insert(0, '.')
import torch
import paper_2001_05585_b200 as T
from paper_2001_05585_b200 import _capi
lib = _capi.load()
dev = torch.device('cuda', 0); st = torch.cuda.current_stream(dev); sp = C.c_void_p(st.cuda_stream)
for n in (1 << 28, 1 << 30):
    xf = T.generate('uniform', 0, n, device=dev, dtype='float32')
    res = torch.zeros(2, dtype=torch.float32, device=dev); ovf = torch.zeros(1, dtype=torch.int32, device=dev)
    for m in (16, 4):
        cfg = T.ReductionConfig(m=m, R=1, B=1024 if m == 16 else 128).to_c()
        fn = lambda: _capi.check(lib.tcr_single_pass_f32_async(C.c_void_p(xf.data_ptr()), n, C.byref(cfg), C.c_void_p(res.data_ptr()), C.c_void_p(ovf.data_ptr()), sp))
        for _ in range(3): fn()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(5): fn()
            b.record(st); b.synchronize(); ts.append(a.elapsed_time(b) / 5)
        t = statistics.median(ts)
        print(f"f32 device m={m} n=2^{n.bit_length()-1}: {t*1e3:.1f} us  {n/t/1e6:.0f} Gelem/s  {4*n/t/1e6:.0f} GB/s  launches {lib.tcr_last_launch_count()}")
    del xf; torch.cuda.empty_cache()
