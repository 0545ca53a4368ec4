#!/usr/bin/env python3
"""Kernel time vs n for the north-star single_pass (AUTO engine), the read probe and the
warp-shuffle comparator: fits
t(n) = a + b n to expose the fixed per-launch cost (pipeline fill, tail, last-CTA finalise).
Profiling tool.   python tools/size_scan.py"""
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2001_05585_b200 as T
    from paper_2001_05585_b200 import _capi
    lib = _capi.load()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    sp = C.c_void_p(st.cuda_stream)
    nmax = 1 << 31
    x = T.generate("uniform", 0, nmax, device=dev)
    res = torch.zeros(2, dtype=torch.float32, device=dev)
    ovf = torch.zeros(1, dtype=torch.int32, device=dev)
    xp, rp, op = C.c_void_p(x.data_ptr()), C.c_void_p(res.data_ptr()), C.c_void_p(ovf.data_ptr())
    cfg = T.ReductionConfig(m=16, R=1, B=1024, finalize=T.Finalize.tree).to_c()

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(reps):
                fn()
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b) / reps * 1e3)
        return statistics.median(ts)

    out = []
    for lg in (24, 26, 27, 28, 29, 30, 31):
        n = 1 << lg
        t_sp = timed(lambda: _capi.check(lib.tcr_single_pass_f16_async(xp, n, C.byref(cfg), rp, op, sp)))
        t_rd = timed(lambda: _capi.check(lib.tcr_read_probe_async(xp, 2 * n, sp)))
        t_sh = timed(lambda: _capi.check(lib.tcr_shuffle_f16_async(xp, n, rp, sp)))
        rec = {"n": n, "single_pass_us": t_sp, "read_probe_us": t_rd, "warp_shuffle_us": t_sh,
               "sp_TBs": 2 * n / t_sp / 1e6, "probe_TBs": 2 * n / t_rd / 1e6, "shuffle_TBs": 2 * n / t_sh / 1e6}
        out.append(rec)
        print(json.dumps(rec), flush=True)
    for key in ("single_pass_us", "read_probe_us", "warp_shuffle_us"):
        a = out[-3]  # 2^29
        b = out[-1]  # 2^31
        slope = (b[key] - a[key]) / (b["n"] - a["n"])
        print(json.dumps({key: {"fixed_us": b[key] - slope * b["n"], "TBs_marginal": 2 / slope / 1e6}}))


if __name__ == "__main__":
    main()
