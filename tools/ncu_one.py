#!/usr/bin/env python3
"""One single_pass launch for ncu captures (profiling tool):
    ncu --set full -k regex:<kernel> -c 1 python tools/ncu_one.py --m 4 --R 1 --B 128 --n 268435456
A warm-up launch first (lazy module load, workspace allocation), then the captured one."""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--R", type=int, default=1)
    ap.add_argument("--B", type=int, default=1024)
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--engine", type=int, default=0)
    ap.add_argument("--f32", action="store_true")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import torch
    import paper_2001_05585_b200 as T
    from paper_2001_05585_b200 import _capi
    lib = _capi.load()
    lib.tcr_enable_profiling_knobs()   # TCR_* profiling knobs from the environment (A/B captures)
    x = T.generate("uniform", 0, a.n, dtype="float32" if a.f32 else "float16")
    res = torch.zeros(2, dtype=torch.float32, device="cuda")
    ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
    cfg = T.ReductionConfig(m=a.m, R=a.R, B=a.B, engine=T.Engine(a.engine), finalize=T.Finalize.tree).to_c()
    fn = lib.tcr_single_pass_f32_async if a.f32 else lib.tcr_single_pass_f16_async
    for _ in range(a.reps):
        _capi.check(fn(C.c_void_p(x.data_ptr()), a.n, C.byref(cfg), C.c_void_p(res.data_ptr()),
                       C.c_void_p(ovf.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    print("value", res[0].item())


if __name__ == "__main__":
    main()
