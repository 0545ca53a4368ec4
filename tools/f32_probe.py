#!/usr/bin/env python3
"""fp32 device-input single_pass throughput (convert on load): m = 16 (register engine with
from_single fused into the load) and m = 4 (convert pass + selector engine).  Profiling tool."""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2001_05585_b200 as T  # noqa: E402
from paper_2001_05585_b200 import _capi  # noqa: E402

lib = _capi.load()
dev = torch.device('cuda', 0)
st = torch.cuda.current_stream(dev)
sp = C.c_void_p(st.cuda_stream)
for n in (1 << 28, 1 << 30):
    xf = T.generate('uniform', 0, n, device=dev, dtype='float32')
    res = torch.zeros(2, dtype=torch.float32, device=dev)
    ovf = torch.zeros(1, dtype=torch.int32, device=dev)
    for m, env in ((16, None), (4, None)):
        if env:
            os.environ[env] = "1"
        cfg = T.ReductionConfig(m=m, R=1, B=1024 if m == 16 else 128, finalize=T.Finalize.tree).to_c()
        fn = lambda: _capi.check(lib.tcr_single_pass_f32_async(C.c_void_p(xf.data_ptr()), n, C.byref(cfg),  # noqa: E731
                                                               C.c_void_p(res.data_ptr()), C.c_void_p(ovf.data_ptr()), sp))
        for _ in range(3):
            fn()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(5):
                fn()
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b) / 5)
        t = statistics.median(ts)
        print(f"f32 device m={m} {env or 'default'} n=2^{n.bit_length()-1}: {t*1e3:.1f} us  {n/t/1e6:.0f} Gelem/s  "
              f"{4*n/t/1e6:.0f} GB/s  value {res[0].item()}", flush=True)
        if env:
            del os.environ[env]
    del xf
    torch.cuda.empty_cache()
