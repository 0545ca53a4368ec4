#!/usr/bin/env python3
"""Interleaved A/B timing of single_pass variants in ONE process on one GPU (profiling tool).

    python tools/ab.py [--n 1073741824] [--rounds 7] [--reps 10] SPEC [SPEC ...]

SPEC = label:engine:R:B[:ENV=VAL,...]  e.g.  async:4:1:1024  tc05:2:1:1024:TCR_DEBUG_MODE=3
(PROBE=1 / SHUFFLE=1 in the ENV list time the streaming-read probe / the warp-shuffle comparator instead, e.g. tma:0:1:1:PROBE=1,TCR_PROBE=tma)
(LIB=path in the ENV list times another build of libtcreduce_b200.so, e.g. a previous commit's;
M=m sets the fragment side, default 16)
Rounds alternate between the specs so clock / thermal drift hits all of them alike; the
median over rounds of the per-round mean kernel time is reported (CUDA events on the
launch stream, inputs 2 GiB > L2).
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _load_other(path):
    import shutil
    import tempfile
    from paper_2001_05585_b200 import _capi
    # a distinct file name so the dynamic loader does not hand back the in-tree library
    tmp = os.path.join(tempfile.mkdtemp(), "libtcr_ab_%d.so" % abs(hash(path)))
    shutil.copy(path, tmp)
    lib = C.CDLL(tmp)
    for name, (res, args) in _capi.SIGNATURES.items():
        if hasattr(lib, name):
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 30)
    ap.add_argument("--rounds", type=int, default=7)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--dist", default="uniform", help="input distribution (generator seed 0 uniform, else seed 1)")
    ap.add_argument("specs", nargs="+")
    a = ap.parse_args()
    import torch
    import paper_2001_05585_b200 as T
    from paper_2001_05585_b200 import _capi
    lib = _capi.load()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    sp = C.c_void_p(st.cuda_stream)
    x = T.generate(a.dist, 0 if a.dist == "uniform" else 1, a.n, device=dev)
    res = torch.zeros(1, dtype=torch.float32, device=dev)
    ovf = torch.zeros(1, dtype=torch.int32, device=dev)
    xp, rp, op = C.c_void_p(x.data_ptr()), C.c_void_p(res.data_ptr()), C.c_void_p(ovf.data_ptr())
    specs = []
    for s in a.specs:
        parts = s.split(":")
        env = dict(kv.split("=") for kv in parts[4].split(",")) if len(parts) > 4 and parts[4] else {}
        lib_path = env.pop("LIB", None)
        m = int(env.pop("M", 16))
        probe = env.pop("PROBE", None) is not None   # time the streaming-read probe instead
        if env.pop("SHUFFLE", None) is not None:     # time the warp-shuffle comparator instead
            probe = "shuffle"
        cfg = T.ReductionConfig(m=m, R=int(parts[2]), B=int(parts[3]), engine=T.Engine(int(parts[1])),
                                finalize=T.Finalize[env.pop("FIN", "tree")])
        specs.append((parts[0], probe if probe else cfg.to_c(), env,
                      _capi.load() if lib_path is None else _load_other(lib_path)))
    times = {s[0]: [] for s in specs}
    vals = {}
    for rnd in range(a.rounds):
        for label, c, env, lib in specs:
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            lib.tcr_enable_profiling_knobs.restype = C.c_int
            lib.tcr_enable_profiling_knobs()   # knobs are read only on this explicit call
            def call():
                if c == "shuffle":
                    _capi.check(lib.tcr_shuffle_f16_async(xp, a.n, rp, sp))
                elif c is True:
                    _capi.check(lib.tcr_read_probe_async(xp, 2 * a.n, sp))
                else:
                    _capi.check(lib.tcr_single_pass_f16_async(xp, a.n, C.byref(c), rp, op, sp))
            try:
                for _ in range(3):
                    call()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(a.reps):
                    call()
                e1.record(st)
                e1.synchronize()
                times[label].append(e0.elapsed_time(e1) / a.reps)
                vals[label] = res.item()
            finally:
                for k, v in old.items():
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
    out = {}
    for label, _, _, _ in specs:
        ms = statistics.median(times[label])
        out[label] = {"ms_median": ms, "ms_min": min(times[label]), "gelem_s": a.n / ms / 1e6,
                      "tb_s": 2 * a.n / ms / 1e9, "value": vals[label]}
        print(f"{label:24s} {ms * 1e3:8.1f} us  {a.n / ms / 1e6:8.1f} Gelem/s  {2 * a.n / ms / 1e9:6.3f} TB/s  "
              f"(min {min(times[label]) * 1e3:.1f} us)  value {vals[label]!r}", flush=True)
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
