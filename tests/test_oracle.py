"""CPU tests: pin the oracle (oracle/tcr_oracle.c) to the reference.

Three anchors, in order of strength:
  1. bit-for-bit equality with the reference headers compiled as-is (oracle/_ref), when built;
  2. the known-answer values of the reference's own tests (test_half.cpp, test_fragment.cpp,
     test_reduction.cpp, acceptance.cpp), restated here with their file:line;
  3. the committed golden fixtures tests/golden/*.json (made by tools/make_goldens.py from _ref).
"""
import json
import math
import os
import struct

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def f32(bits):
    return struct.unpack("<f", struct.pack("<I", bits))[0]


# ----------------------------------------------------------------- 2. reference known answers

def test_half_kats(oracle):  # test_half.cpp:22-53
    O = oracle
    assert O.to_single(O.from_single(1.0)) == 1.0
    assert O.from_single(1.0) == 0x3C00
    assert O.to_single(O.from_single(0.1)) == 0.0999755859375
    assert math.isinf(O.to_single(O.from_single(65520.0)))
    assert O.to_single(O.from_single(65519.0)) == 65504.0
    assert O.from_single(-0.0) == 0x8000
    assert O.from_single(float("inf")) == 0x7C00
    assert O.from_single(float("-inf")) == 0xFC00
    assert O.from_single(float("nan")) == 0x7E00
    assert O.from_single(f32(0xFFC00123)) == 0x7E00
    assert O.to_single(0x7BFF) == 65504.0
    assert O.to_single(0x0001) == 5.9604644775390625e-8


def test_half_roundtrip_and_decode_all_patterns(oracle):  # test_half.cpp:55-104; acceptance crit 8
    O = oracle
    bits = np.arange(0x10000, dtype=np.uint32)
    vals = np.array([O.to_single(int(b)) for b in bits], np.float32)
    ref = np.arange(0x10000, dtype=np.uint16).view(np.float16).astype(np.float32)  # IEEE decode
    same = (vals.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(vals) & np.isnan(ref))
    assert same.all()
    finite = (bits & 0x7C00) != 0x7C00
    back = np.array([O.from_single(float(v)) for v in vals[finite]], np.uint32)
    assert (back == bits[finite]).all()


def test_from_single_matches_ieee_rne(oracle):  # test_half.cpp:74-92 (nearest-value reference)
    O = oracle
    rng = np.random.default_rng(0xC0FFEE)
    xs = rng.integers(0, 2**32, 20000, dtype=np.uint64).astype(np.uint32).view(np.float32)
    xs = xs[~np.isnan(xs)]
    mine = np.array([O.from_single(float(v)) for v in xs], np.uint16)
    ieee = xs.astype(np.float16).view(np.uint16)  # numpy: IEEE round-to-nearest-even
    assert (mine == ieee).all()


def test_generator_reproducible_and_jump_ahead(oracle):  # test_harness.cpp:12-55
    O = oracle
    for dist, seed in (("uniform", 99), ("normal", 12345), ("integers", 4)):
        a = O.generate(dist, seed, 20001, lo=-3, hi=7)
        assert np.array_equal(a, O.generate(dist, seed, 20001, lo=-3, hi=7))
        tail = O.generate(dist, seed, 5000, lo=-3, hi=7, first=7777)
        assert np.array_equal(a[7777:12777].view(np.uint32), tail.view(np.uint32))
    u = O.generate("uniform", 99, 100000)
    assert (u >= 0).all() and (u < 1).all() or (u <= 1).all()
    i = O.generate("integers", 4, 50000, lo=-3, hi=7)
    assert i.min() >= -3 and i.max() <= 7 and (i == np.floor(i)).all()
    z = O.generate("normal", 7, 1000000)
    assert abs(z.astype(np.float64).mean()) < 5.0 / 1000.0
    assert abs(z.astype(np.float64).var() - 1.0) < 0.01


def test_chain_kats(oracle):  # test_reduction.cpp:85-101
    O = oracle
    v, ov, mc = O.chained_warp_reduce(np.ones(32, np.float32), 0, m=4, R=2)
    assert v == 32.0
    seq = np.arange(1, 33, dtype=np.float32)
    assert O.chained_warp_reduce(seq, 0, m=4, R=2)[0] == 528.0
    v, ov, mc = O.chained_warp_reduce(seq, 0, m=4, R=1)
    assert v == 136.0 and mc == 2
    with pytest.raises(IndexError):
        O.chained_warp_reduce(seq, 17, m=4, R=1)


def test_single_pass_kats(oracle):  # test_reduction.cpp:119-135
    O = oracle
    out = O.single_pass(np.ones(2048, np.float32), m=4, R=4, B=128)
    assert out.value == 2048.0 and out.atomic_count == 8 and out.mma_count == 8 * 4 * 5
    assert O.single_pass(np.arange(1, 17, dtype=np.float32), m=4, R=1, B=32).value == 136.0
    u = O.generate("uniform", 0, 1000000)
    uo = O.single_pass(u, m=4, R=4, B=128)
    assert not uo.overflow
    ref = O.oracle64(u)
    assert abs(uo.value - ref) / abs(ref) * 100 < 0.001


def test_integer_exactness_and_order_invariance(oracle):  # test_reduction.cpp:155-176; acceptance crit 5
    O = oracle
    for seed in (0, 1, 2):
        ints = O.generate("integers", seed, 100000)
        ref = O.oracle64(ints)
        assert O.single_pass(ints, m=4, R=4, B=128).value == ref
        assert O.single_pass(ints, m=16, R=1, B=1024).value == ref
    ints = O.generate("integers", 9, 200000)
    asc = O.single_pass(ints, m=4, R=4, B=128).value
    for s in (1, 2, 3):
        assert O.single_pass(ints, m=4, R=4, B=128, atomic_order=1, atomic_seed=s).value == asc


def test_zero_padding_neutral(oracle):  # test_reduction.cpp:178-189
    O = oracle
    base = O.generate("normal", 17, 5000)
    padded = np.concatenate([base, np.zeros(333, np.float32)])
    for v, kw in (("shuffle32", {}), ("half_tree", {}), ("recurrence", dict(m=4, R=5, B=32)),
                  ("single_pass", dict(m=4, R=4, B=128))):
        assert O.reduce(base, variant=v, **kw).value == O.reduce(padded, variant=v, **kw).value


def test_validation(oracle):  # test_reduction.cpp:221-234
    O = oracle
    for bad in (dict(B=48), dict(B=2048), dict(R=0), dict(f=1.5), dict(m=3), dict(m=1)):
        cfg = O.make_config(**{**dict(m=4, R=1, B=128, f=0.5), **bad})
        assert O.lib().orc_validate(cfg) == -1
    with pytest.raises(ValueError):
        O.reduce(np.zeros(0, np.float32), variant="shuffle32")


def test_thread_count_invariance(oracle):
    O = oracle
    x = O.generate("uniform", 5, 300007)
    a, ba = O.single_pass(x, threads=1, want_blocks=True, m=16, R=3, B=96)
    b, bb = O.single_pass(x, threads=7, want_blocks=True, m=16, R=3, B=96)
    assert a.as_dict() == b.as_dict() and np.array_equal(ba.view(np.uint32), bb.view(np.uint32))
    h = np.array([O.from_single(float(v)) for v in x], np.uint16)
    c = O.single_pass(h, threads=3, m=16, R=3, B=96)
    assert c.as_dict() == a.as_dict()


# ----------------------------------------------------------------- 1. bit-for-bit vs the reference

needs_ref = pytest.mark.skipif(not __import__("oracle").ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("variant", ["oracle64", "shuffle32", "half_tree", "recurrence", "single_pass", "split"])
def test_oracle_equals_reference_all_variants(oracle, variant):
    O = oracle
    rng = np.random.default_rng(1)
    for dist, seed, n in (("uniform", 0, 70001), ("normal", 3, 65536), ("integers", 2, 40000)):
        x = O.generate(dist, seed, n)
        for (m, R, B, f) in ((4, 1, 128, 0.5), (16, 1, 1024, 0.3), (16, 4, 128, 1.0), (8, 3, 96, 0.0),
                             (2, 7, 64, 0.9), (32, 2, 64, 0.5)):
            a = O.reduce(x, variant=variant, m=m, R=R, B=B, f=f).as_dict()
            b = O.ref_reduce(x, variant=variant, m=m, R=R, B=B, f=f).as_dict()
            assert a == b, (dist, m, R, B, a, b)
    assert rng is not None


@needs_ref
def test_oracle_generator_equals_reference(oracle):
    O = oracle
    for dist, seed in (("uniform", 0), ("normal", 1), ("integers", 2), ("constant", 0)):
        a = O.generate(dist, seed, 100001)
        b = O.ref_generate(dist, seed, 100001)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@needs_ref
def test_parallel_reference_is_bit_identical(oracle):  # SURVEY Appendix A restatement
    O = oracle
    x = O.generate("uniform", 3, (1 << 20) + 7)
    a = O.ref_reduce(x, variant="single_pass", m=16, R=1, B=1024)
    b = O.ref_single_pass_parallel(x, 4, m=16, R=1, B=1024)
    assert a.as_dict() == b.as_dict()


# ----------------------------------------------------------------- 3. committed golden fixtures

def _golden(name):
    p = os.path.join(GOLDEN, name)
    if not os.path.exists(p):
        pytest.skip(f"{name} not generated")
    return json.load(open(p))


def test_oracle_matches_golden_small(oracle):
    O = oracle
    g = _golden("reference_small.json")
    cache = {}
    for case in g["cases"]:
        if case["dist"] is None:
            continue
        key = (case["dist"], case["seed"], case["n"])
        if key not in cache:
            cache[key] = O.generate(case["dist"], case["seed"], case["n"])
        cfg = {k: case[k] for k in ("m", "R", "B") if k in case}
        cfg.update({k: case[k] for k in ("atomic_order", "atomic_seed") if k in case})
        out = O.single_pass(cache[key], threads=4, **cfg)
        exp = case["outcome"]
        assert out.value == exp["value"] or (math.isnan(out.value) and math.isnan(exp["value"])), case["tag"]
        assert bool(out.overflow) == exp["overflow"]
        for k in ("atomic_count", "mma_count", "shuffle_count", "sim_steps", "level_count"):
            assert getattr(out, k) == exp[k], (case["tag"], k)


def test_generator_matches_golden(oracle):
    O = oracle
    g = _golden("reference_small.json")
    import hashlib
    for rec in g["generator"]:
        x = O.generate(rec["dist"], rec["seed"], rec["n"], lo=rec["lo"], hi=rec["hi"])
        assert hashlib.sha256(x.tobytes()).hexdigest() == rec["sha256_f32"]
        h = O.generate_f16(rec["dist"], rec["seed"], 4096, lo=rec["lo"], hi=rec["hi"])
        assert hashlib.sha256(h.tobytes()).hexdigest() == rec["sha256_f16_first4096"]


def test_survey_measured_goldens(oracle):
    """m=16 integer sweep values and the uniform 2^20 cfg1 values."""
    O = oracle
    expect = {0: 4715354.0, 1: 4716649.0, 2: 4718742.0}
    for seed, val in expect.items():
        x = O.generate("integers", seed, 1 << 20)
        assert O.single_pass(x, threads=4, m=16, R=1, B=1024).value == val
    u = O.generate("uniform", 0, 1 << 20)
    assert O.oracle64(u) == 524199.35321258294
    h = O.generate_f16("uniform", 0, 1 << 20)
    assert O.exact_sum_f16(h)[0] == 524199.3321583271
    assert O.single_pass(u, m=16, R=1, B=1024).value == 524199.0
    assert O.single_pass(u, m=4, R=4, B=128).value == 524198.625
