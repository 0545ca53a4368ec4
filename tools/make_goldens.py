"""Generate tests/golden/*.json from the reference itself (oracle/_ref) and the pinned oracle.

Run in the build container (needs /root/reference to have built oracle/_ref):
    python tools/make_goldens.py [--large] [--huge]

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


# BASELINE configs[2] grid (every (R, B) of the paper's sweep) and the configs[3] precision-study
# points; every (dist, seed, n) of the study carries the four study configs.
SWEEP_RB = [(R, B) for B in (32, 128, 256, 512, 1024) for R in (1, 2, 3, 4, 5)]
STUDY_RB = [(1, 1024), (4, 128), (1, 128), (5, 32)]


def gen_f16(dist: str, seed: int, first: int, n: int, threads: int) -> np.ndarray:
    """Elements [first, first+n) of generate(dist, seed) rounded to binary16, in parallel slices
    (the jump-ahead generator is position-independent: harness.hpp:47-80)."""
    from concurrent.futures import ThreadPoolExecutor
    h = np.empty(n, np.uint16)
    step = -(-n // threads)
    step += (-step) % 2          # normal pairs never straddle a slice
    def run(i):
        a = i * step
        b = min(n, a + step)
        if a < b:
            O._check(O.lib().orc_generate_range_f16(O.DISTS[dist], seed, 0, 9, 1.0, first + a, b - a, h[a:b]))
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, range(threads)))
    return h


def large(threads: int) -> dict:
    lg: dict = {"source": "oracle/liboracle.so (bit-identical restatement, re-pinned below)", "cases": []}
    # re-pin the restatement against the reference at 2^24 with the reference's parallel form
    for dist, seed, (m, R, B) in (("normal", 3, (16, 4, 128)), ("uniform", 0, (16, 1, 1024)),
                                  ("uniform", 5, (16, 3, 256))):
        x = O.ref_generate(dist, seed, (1 << 24) + 12345)
        a, ab = O.single_pass(x, threads=threads, want_blocks=True, m=m, R=R, B=B)
        b, bb = O.ref_single_pass_parallel(x, threads, want_blocks=True, m=m, R=R, B=B)
        assert a.as_dict() == b.as_dict(), (a.as_dict(), b.as_dict())
        assert np.array_equal(ab.view(np.uint32), bb.view(np.uint32))
        lg.setdefault("repins", []).append({"n": int(x.size), "dist": dist, "seed": seed, "m": m, "R": R, "B": B,
                                            "value": a.value})
    lg["repin"] = lg["repins"][0]
    del x
    for dist, seed in (("uniform", 0), ("normal", 1), ("normal", 2), ("normal", 3)):
        for lgn in (26, 27, 28, 29, 30):
            n = 1 << lgn
            t = time.time()
            x = O.generate(dist, seed, n)
            o64 = O.oracle64(x)
            del x
            h = gen_f16(dist, seed, 0, n, threads)
            ex, ab = O.exact_sum_f16(h)
            rec = {"dist": dist, "seed": seed, "n": n, "oracle64_f32_input": o64, "exact_f16_sum": ex,
                   "abs_f16_sum": ab, "single_pass": {}}
            pts = list(STUDY_RB)
            if dist == "uniform" and lgn == 28:
                pts += [rb for rb in SWEEP_RB if rb not in pts]
            for (R, B) in pts:
                o, blocks = O.single_pass(h, threads=threads, want_blocks=True, m=16, R=R, B=B)
                d = outcome(o)
                d["blocks_sha256"] = sha(blocks)
                rec["single_pass"][f"m16_R{R}_B{B}"] = d
            lg["cases"].append(rec)
            print(dist, seed, n, len(pts), f"{time.time() - t:.1f}s", flush=True)
            del h
    return lg


def huge(threads: int, lgn: int = 34, chunk_lg: int = 28) -> dict:
    """BASELINE configs[4]: uniform s0, n = 2^34 (32 GiB of binary16), streamed through the
    restatement in 2^28-element slices (whole blocks each: the block partition is global).
    The value is the reference's serial ascending fp32 sum of the block results
    (reduction.hpp:264-268), accumulated across slices in block order."""
    from fractions import Fraction
    n = 1 << lgn
    out: dict = {"source": "oracle/liboracle.so streamed (blocks of every 2^%d slice, serial fp32 combine)" % chunk_lg,
                 "dist": "uniform", "seed": 0, "n": n, "single_pass": {}}
    cfgs = [(16, 1, 1024)]
    accs = {c: np.float32(0.0) for c in cfgs}
    hashes = {c: hashlib.sha256() for c in cfgs}
    counts = {c: 0 for c in cfgs}
    ovf = {c: False for c in cfgs}
    exact = Fraction(0)
    absum = Fraction(0)
    t = time.time()
    for s in range(n >> chunk_lg):
        h = gen_f16("uniform", 0, s << chunk_lg, 1 << chunk_lg, threads)
        e, a = O.exact_sum_f16(h)      # exact in binary64 at 2^28 elements (< 2^53 units of 2^-24)
        exact += Fraction(e)
        absum += Fraction(a)
        for c in cfgs:
            m, R, B = c
            o, blocks = O.single_pass(h, threads=threads, want_blocks=True, m=m, R=R, B=B)
            # np.add.accumulate is a strictly sequential fp32 running sum (no pairwise blocking)
            seq = np.concatenate([np.array([accs[c]], np.float32), blocks])
            accs[c] = np.add.accumulate(seq, dtype=np.float32)[-1]
            hashes[c].update(blocks.tobytes())
            counts[c] += blocks.size
            ovf[c] = ovf[c] or bool(o.overflow)
        if s % 8 == 0:
            print(f"slice {s}/{n >> chunk_lg} {time.time() - t:.0f}s", flush=True)
    out["exact_f16_sum"] = float(exact)
    out["abs_f16_sum"] = float(absum)
    for c in cfgs:
        m, R, B = c
        out["single_pass"][f"m{m}_R{R}_B{B}"] = {"value": float(accs[c]), "overflow": ovf[c], "blocks": counts[c],
                                                 "blocks_sha256": hashes[c].hexdigest()}
    out["seconds"] = time.time() - t
    return out


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
    if "--huge" in sys.argv:
        hg = huge(os.cpu_count() or 1)
        with open(os.path.join(OUT, "oracle_2e34.json"), "w") as f:
            json.dump(hg, f, indent=1)


if __name__ == "__main__":
    main()
