#!/usr/bin/env python3
"""ORDERED single_pass phase timing (profiling tool):
    python tools/ordered_one.py [m:R:B:lgn[:order] ...]   (order 1 = seeded permutation, seed 3)
Prints the walk counters and the %globaltimer phases of the ascending ORDERED kernel."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2001_05585_b200 as T  # noqa: E402
from paper_2001_05585_b200 import _capi  # noqa: E402

lib = _capi.load()
specs = sys.argv[1:] or ["16:1:1024:30", "16:4:128:30", "4:1:128:28", "4:1:128:30", "16:1:1024:30:1", "4:1:128:28:1"]
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for spec in specs:
    m, R, B, lgn, *rest = map(int, spec.split(":"))
    order = rest[0] if rest else 0
    n = 1 << lgn
    x = T.generate("uniform", 0, n)
    res = torch.zeros(2, dtype=torch.float32, device="cuda")
    ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
    cfg = T.ReductionConfig(m=m, R=R, B=B, finalize=T.Finalize.ordered, atomic_order=T.AtomicOrder(order),
                            atomic_seed=3).to_c()
    st = (C.c_ulonglong * 9)()
    for _ in range(3):
        _capi.check(lib.tcr_single_pass_f16_async(C.c_void_p(x.data_ptr()), n, C.byref(cfg), C.c_void_p(res.data_ptr()),
                                                  C.c_void_p(ovf.data_ptr()), sp))
        torch.cuda.synchronize()
        lib.tcr_ordered_stats(st)
    t0 = st[4]
    print(f"m={m} R={R} B={B} n=2^{lgn} order={order}: value {res[0].item()} walk: tree nodes {st[0]} CTA runs {st[1]} "
          f"segment records {st[2]} serial segments {st[3]} | us: lookback {(st[5]-t0)/1e3:.1f} "
          f"records {(st[6]-t0)/1e3:.1f} walk start {(st[7]-t0)/1e3:.1f} end {(st[8]-t0)/1e3:.1f}", flush=True)
    del x
    torch.cuda.empty_cache()
