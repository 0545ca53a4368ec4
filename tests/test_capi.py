"""CPU tests of the C ABI boundary: the library loads, exports every symbol the header
declares, and its host-side logic (validation, counters, geometry) mirrors the reference.
No kernel is launched here."""
import ctypes as C

import numpy as np
import pytest

import paper_2001_05585_b200 as T
from paper_2001_05585_b200 import _capi


def test_library_exports_every_header_symbol():
    lib = _capi.load()
    syms = _capi.header_symbols()
    assert len(syms) >= 22
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_capi.SIGNATURES) == set(syms)


def test_config_defaults_match_reference():  # reduction.hpp:40-46
    c = _capi.tcr_config()
    _capi.load().tcr_config_init(C.byref(c))
    assert (c.variant, c.m, c.R, c.B, c.f, c.atomic_order, c.atomic_seed) == (4, 4, 1, 128, 0.5, 0, 0)
    d = T.ReductionConfig()
    assert (d.variant, d.m, d.R, d.B, d.f) == (T.Variant.single_pass, 4, 1, 128, 0.5)


@pytest.mark.parametrize("bad", [dict(B=48), dict(B=2048), dict(B=0), dict(R=0), dict(f=1.5), dict(f=-0.1),
                                 dict(m=3), dict(m=1), dict(m=0)])
def test_validate_mirrors_reference(bad, oracle):  # reduction.hpp:50-56, fragment.hpp:22-25
    cfg = T.ReductionConfig(**bad)
    with pytest.raises(ValueError):
        cfg.validate()
    ocfg = oracle.make_config(**{**dict(m=4, R=1, B=128, f=0.5), **bad})
    assert oracle.lib().orc_validate(ocfg) == -1


def test_validate_accepts_reference_grid():
    for m in (2, 4, 8, 16, 32, 64):
        for B in range(32, 1025, 32):
            T.ReductionConfig(m=m, B=B, R=3).validate()


@pytest.mark.parametrize("n", [1, 15, 16, 2048, 100003, 1 << 20, (1 << 30) + 1])
@pytest.mark.parametrize("m,R,B", [(16, 1, 1024), (16, 4, 128), (16, 5, 96), (4, 4, 128), (8, 3, 32)])
def test_counters_follow_reference_formulas(n, m, R, B, oracle):  # reduction.hpp:240-273
    ours = T.counters(n, T.ReductionConfig(m=m, R=R, B=B))
    if n <= 200000:
        x = np.ones(n, np.float32)
        ref = oracle.single_pass(x, threads=4, m=m, R=R, B=B)
        for k in ("level_count", "sim_steps", "mma_count", "atomic_count", "shuffle_count"):
            assert getattr(ours, k) == getattr(ref, k), k
    blocks = max(1, -(-n // (R * m * m * (B // 32))))
    assert ours.atomic_count == blocks
    assert ours.mma_count == blocks * (B // 32) * (R + 1)
    assert T.block_count(n, T.ReductionConfig(m=m, R=R, B=B)) == blocks


def test_reference_pinned_counter_example():  # test_reduction.cpp:121-124
    o = T.counters(2048, T.ReductionConfig(m=4, R=4, B=128))
    assert o.atomic_count == 8 and o.mma_count == 160


def test_empty_input_is_invalid_argument():  # reduction.hpp:282
    with pytest.raises(ValueError):
        T.reduce(np.zeros(0, np.float32), T.ReductionConfig(m=16))
