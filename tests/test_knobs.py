"""Profiling knobs are never read implicitly (CPU: the geometry is host code).  The reference is a
pure function of input and config (reduction.hpp:19-21); the group size G -- and with it the
TREE order and the shard alignment -- must not move with the environment unless a profiling
tool explicitly asks (tcr_enable_profiling_knobs)."""
import ctypes as C

import paper_2001_05585_b200 as T
from paper_2001_05585_b200 import _capi


def _ge(cfg):
    c = cfg.to_c()
    return _capi.load().tcr_group_elems(C.byref(c))


def test_environment_is_ignored_without_explicit_opt_in(monkeypatch):
    cfg = T.ReductionConfig(m=16, R=1, B=1024)
    base = _ge(cfg)
    monkeypatch.setenv("TCR_GROUP_TARGET", "4096")
    assert _ge(cfg) == base
    with _capi.profiling_knobs({"TCR_GROUP_TARGET": "4096"}):   # G = 1 block
        assert _ge(cfg) != base
    assert _ge(cfg) == base


def test_group_cap_knob_cannot_exceed_the_chunk_table():
    # a cap beyond the engine's shared-memory chunk table (1024 chunks at m = 16) is clamped:
    # G * W never exceeds it
    cfg = T.ReductionConfig(m=16, R=1, B=1024)     # W = 32 chunks per block
    with _capi.profiling_knobs({"TCR_GROUP_TARGET": str(1 << 30), "TCR_GROUP_CAP": "1000000"}):
        ge = _ge(cfg)
    chunk = 16 * 16 * 1
    assert ge // chunk <= 1024
