import ctypes as C, torch, statistics, sys, os
sys.path.insert(0, os.getcwd())
import paper_2001_05585_b200 as T
from paper_2001_05585_b200 import _capi
lib = _capi.load()
st = torch.cuda.current_stream(); sp = C.c_void_p(st.cuda_stream)
for (m, R, B, n) in ((16, 1, 1024, 1 << 30), (16, 4, 128, 1 << 30), (4, 1, 128, 1 << 28), (4, 1, 128, 1 << 30), (4, 4, 128, 1 << 30)):
    for dist in ("uniform", "normal"):
        x = T.generate(dist, 0 if dist == "uniform" else 1, n)
        res = torch.zeros(2, dtype=torch.float32, device="cuda"); ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
        for fin, order in ((0, 0), (1, 0), (1, 1)):
            cfg = T.ReductionConfig(m=m, R=R, B=B, finalize=T.Finalize(fin), atomic_order=T.AtomicOrder(order), atomic_seed=3).to_c()
            f = lambda: _capi.check(lib.tcr_single_pass_f16_async(C.c_void_p(x.data_ptr()), n, C.byref(cfg), C.c_void_p(res.data_ptr()), C.c_void_p(ovf.data_ptr()), sp))
            for _ in range(2): f()
            ts = []
            for _ in range(7):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st); f(); b.record(st); b.synchronize(); ts.append(a.elapsed_time(b))
            print(f"{dist:8s} m={m} R={R} B={B} n=2^{n.bit_length()-1} finalize={['tree','ordered'][fin]} order={['ascending','seeded'][order]}: {statistics.median(ts)*1e3:.1f} us value {res[0].item()}", flush=True)
        del x; torch.cuda.empty_cache()
