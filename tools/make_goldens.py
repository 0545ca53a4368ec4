"""Generate tests/golden/*.json from the reference itself (oracle/_ref) and the pinned oracle.

Run in the build container (needs /root/reference to have built oracle/_ref):
    python tools/make_goldens.py [--large]

Small cases come straight from the UNMODIFIED reference compiled by oracle/Makefile
(tcreduce::single_pass_reduce, generate, from_single).  Large cases (n = 2^26 .. 2^30) use the
C restatement oracle/liboracle.so with all host threads; tests/test_oracle.py pins that
restatement bit-for-bit against the reference on every small case first, and this script
re-checks it against the reference at 2^24 before trusting it at 2^30.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(o) -> dict:
    d = o.as_dict()
    d["overflow"] = bool(d["overflow"])
    return d


def small() -> dict:
    assert O.ref_available(), "oracle/_ref not built (needs /root/reference)"
    g: dict = {"source": "oracle/_ref/libtcreduce_ref.so = reference headers compiled as-is", "cases": []}

    # generator fingerprints (harness.hpp:47-80)
    g["generator"] = []
    for dist, seed, lo, hi in [("uniform", 0, 0, 9), ("uniform", 3, 0, 9), ("normal", 1, 0, 9), ("normal", 17, 0, 9),
                               ("integers", 0, 0, 9), ("integers", 4, -3, 7)]:
        x = O.ref_generate(dist, seed, 65537, lo=lo, hi=hi)
        h = np.array([O.ref().ref_from_single(float(v)) for v in x[:4096]], np.uint16)
        g["generator"].append({"dist": dist, "seed": seed, "lo": lo, "hi": hi, "n": 65537,
                               "first8_f32_bits": [int(v) for v in x[:8].view(np.uint32)],
                               "sha256_f32": sha(x), "sha256_f16_first4096": sha(h)})

    def case(tag, x, dist=None, seed=None, **cfg):
        o = O.ref_reduce(x, variant="single_pass", **cfg)
        rec = {"tag": tag, "n": int(x.size), "dist": dist, "seed": seed, **cfg, "outcome": outcome(o),
               "oracle64": O.ref().ref_oracle64(x, x.size)}
        g["cases"].append(rec)

    # reference unit-test inputs (test_reduction.cpp:119-135, :155-189)
    case("ones2048_R4_B128", np.ones(2048, np.float32), m=4, R=4, B=128)
    case("iota16_R1_B32", np.arange(1, 17, dtype=np.float32), m=4, R=1, B=32)
    case("iota16_m16", np.arange(1, 17, dtype=np.float32), m=16, R=1, B=32)
    for seed in (0, 1, 2):
        x = O.ref_generate("integers", seed, 1 << 20)
        for B in (32, 128, 256, 512, 1024):
            for R in (1, 2, 3, 4, 5):
                case(f"int_s{seed}_m16_R{R}_B{B}", x, "integers", seed, m=16, R=R, B=B)
        case(f"int_s{seed}_m4_R4_B128", x, "integers", seed, m=4, R=4, B=128)
    for dist, seed in (("uniform", 0), ("normal", 1), ("normal", 17)):
        x = O.ref_generate(dist, seed, 1 << 20)
        for (m, R, B) in ((16, 1, 1024), (16, 4, 128), (16, 2, 32), (16, 5, 96), (4, 1, 1024), (4, 4, 128)):
            case(f"{dist}_s{seed}_m{m}_R{R}_B{B}", x, dist, seed, m=m, R=R, B=B)
        for s in (1, 2, 3):
            case(f"{dist}_s{seed}_m16_R1_B1024_perm{s}", x, dist, seed, m=16, R=1, B=1024, atomic_order=1,
                 atomic_seed=s)
    # ragged sizes and zero padding
    x = O.ref_generate("uniform", 11, 100003)
    for (m, R, B) in ((16, 1, 1024), (16, 3, 64), (16, 4, 128)):
        case(f"uniform_s11_ragged_m{m}_R{R}_B{B}", x, "uniform", 11, m=m, R=R, B=B)
    # overflow: values whose column sums pass 65504 (C_R -> inf)
    case("overflow_const_8192", np.full(1 << 16, 8192.0, np.float32), m=16, R=1, B=128)
    return g


def large(threads: int) -> dict:
    lg: dict = {"source": "oracle/liboracle.so (bit-identical restatement, re-pinned below)", "cases": []}
    # re-pin the restatement against the reference at 2^24 with the reference's parallel form
    x = O.ref_generate("normal", 3, (1 << 24) + 12345)
    a = O.single_pass(x, threads=threads, m=16, R=4, B=128)
    b = O.ref_single_pass_parallel(x, threads, m=16, R=4, B=128)
    assert a.as_dict() == b.as_dict(), (a.as_dict(), b.as_dict())
    lg["repin"] = {"n": int(x.size), "dist": "normal", "seed": 3, "m": 16, "R": 4, "B": 128, "value": a.value}
    del x
    for dist, seed in (("uniform", 0), ("normal", 1), ("normal", 2), ("normal", 3)):
        for lgn in (26, 28, 30):
            if dist != "uniform" and seed != 1 and lgn != 26:
                continue
            n = 1 << lgn
            t = time.time()
            x = O.generate(dist, seed, n)
            o64 = O.oracle64(x)
            h = np.empty(n, np.uint16)
            O.lib().orc_generate_range_f16(O.DISTS[dist], seed, 0, 9, 1.0, 0, n, h)
            del x
            ex, ab = O.exact_sum_f16(h)
            rec = {"dist": dist, "seed": seed, "n": n, "oracle64_f32_input": o64, "exact_f16_sum": ex,
                   "abs_f16_sum": ab, "single_pass": {}}
            for (m, R, B) in ((16, 1, 1024), (16, 4, 128), (16, 1, 128), (16, 5, 32)):
                o = O.single_pass(h, threads=threads, m=m, R=R, B=B)
                rec["single_pass"][f"m{m}_R{R}_B{B}"] = outcome(o)
            lg["cases"].append(rec)
            print(dist, seed, n, f"{time.time() - t:.1f}s", flush=True)
            del h
    return lg


def main():
    os.makedirs(OUT, exist_ok=True)
    O.build()
    g = small()
    with open(os.path.join(OUT, "reference_small.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("small cases:", len(g["cases"]))
    if "--large" in sys.argv:
        lg = large(os.cpu_count() or 1)
        with open(os.path.join(OUT, "oracle_large.json"), "w") as f:
            json.dump(lg, f, indent=1)


if __name__ == "__main__":
    main()
