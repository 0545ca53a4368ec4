#!/usr/bin/env python3
"""Interleaved A/B of the fp32 device-input path between this build and another library
(LIB=path).  Profiling tool:  python tools/f32_ab.py build/ab/other.so"""
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2001_05585_b200 as T  # noqa: E402
from ab import _load_other  # noqa: E402
from paper_2001_05585_b200 import _capi  # noqa: E402


def main():
    libs = {"new": _capi.load(), "old": _load_other(sys.argv[1])}
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    for n in (1 << 28, 1 << 30):
        xf = T.generate("uniform", 0, n, device=dev, dtype="float32")
        res = torch.zeros(2, dtype=torch.float32, device=dev)
        ovf = torch.zeros(1, dtype=torch.int32, device=dev)
        for m, R, B in ((16, 1, 1024), (16, 4, 128), (4, 1, 128), (4, 1, 1024)):
            cfg = T.ReductionConfig(m=m, R=R, B=B, finalize=T.Finalize.tree).to_c()
            t = {k: [] for k in libs}
            for _ in range(5):
                for name, lib in libs.items():
                    fn = lambda: lib.tcr_single_pass_f32_async(C.c_void_p(xf.data_ptr()), n, C.byref(cfg),  # noqa: E731
                                                               C.c_void_p(res.data_ptr()), C.c_void_p(ovf.data_ptr()),
                                                               C.c_void_p(st.cuda_stream))
                    fn()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(st)
                    for _ in range(5):
                        fn()
                    b.record(st)
                    b.synchronize()
                    t[name].append(a.elapsed_time(b) / 5)
            for name in libs:
                ms = statistics.median(t[name])
                print(f"n=2^{n.bit_length()-1} m={m} R={R} B={B} {name}: {ms*1e3:.1f} us {4*n/ms/1e6:.0f} GB/s value {res[0].item()}",
                      flush=True)
        del xf
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
