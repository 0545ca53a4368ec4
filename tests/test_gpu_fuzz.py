"""Randomised parity sweep (fixed seed): random fragment side, chain length, block size, length,
finalize order, engine, variant and input distribution, each reduced on the B200 through the C
ABI and checked against the reference restatement (oracle/, the checker only).  Catches the
combinations the structured tests do not enumerate."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2001_05585_b200 as T  # noqa: E402

DEV = "cuda"
CASES = 500


def _case(rng):
    m = int(rng.choice([2, 4, 4, 8, 16, 16, 16, 32, 64, 128, 256, 512, 1024]))
    R = int(rng.choice([1, 1, 2, 3, 4, 5, 6, 7, 8, 9, 12]))
    B = 32 * int(rng.integers(1, 33))
    if m >= 256:
        R = min(R, 2)
    n = int(rng.choice([1, 7, 255, 4096, 65537, 300_001, 1 << 20, (1 << 21) + 13]))
    dist = str(rng.choice(["uniform", "normal", "integers"]))
    seed = int(rng.integers(0, 1000))
    fin = T.Finalize(int(rng.integers(0, 3)))
    engine = T.Engine(int(rng.choice([0, 0, 1, 2, 3, 4]))) if m == 16 else T.Engine.auto
    variant = str(rng.choice(["single_pass"] * 6 + ["recurrence", "split", "shuffle32", "half_tree", "oracle64"]))
    return m, R, B, n, dist, seed, fin, engine, variant


@pytest.fixture(scope="module")
def oracle():
    import oracle as O
    O.lib()
    return O


@pytest.mark.parametrize("k", range(CASES))
def test_random_config_matches_reference(oracle, k):
    rng = np.random.default_rng(1000 + k)
    m, R, B, n, dist, seed, fin, engine, variant = _case(rng)
    if dist == "integers":
        x = oracle.generate("integers", seed, n)
    else:
        x = oracle.generate(dist, seed, n)
    h = x.astype(np.float16).view(np.uint16)
    xd = torch.from_numpy(h.view(np.int16).copy()).to(DEV).view(torch.float16)
    cfg = T.ReductionConfig(variant=T.Variant[variant], m=m, R=R, B=B, f=float(rng.random()), finalize=fin,
                            engine=engine)
    got = T.reduce(xd, cfg)
    ref = oracle.reduce(h.view(np.float16).astype(np.float32), variant=variant, m=m, R=R, B=B, f=cfg.f)
    tag = (m, R, B, n, dist, seed, fin.name, engine.name, variant)
    # counters follow the reference formulas exactly (the device is a different schedule, the
    # simulated grid is the same)
    assert got.level_count == ref.level_count and got.mma_count == ref.mma_count, tag
    assert got.atomic_count == ref.atomic_count and got.shuffle_count == ref.shuffle_count, tag
    if not np.isfinite(ref.value) or ref.overflow:
        assert got.overflow, tag
        return
    assert not got.overflow, tag
    exact, absum = oracle.exact_sum_f16(h)
    if variant == "single_pass" and fin == T.Finalize.ordered:
        # ORDERED is the reference's own combine: wherever the block results are bit-identical
        # the value must be too (reduction.hpp:257-268)
        _, ref_blocks = oracle.single_pass(h, threads=4, want_blocks=True, m=m, R=R, B=B)
        gb = T.block_results(xd, T.ReductionConfig(m=m, R=R, B=B, engine=engine)).cpu().numpy()
        if np.array_equal(gb.view(np.uint32), ref_blocks.view(np.uint32)):
            assert got.value == ref.value, (tag, got.value, ref.value)
    if variant in ("shuffle32", "half_tree", "oracle64"):
        assert got.value == ref.value, tag                     # bit-exact strided trees / serial binary64
    elif dist == "integers" and 9 * R * m <= 2048 and absum < 2 ** 24:
        assert got.value == ref.value, tag                     # exact integer sums
    else:
        # different (fixed) combine order and tensor-core inner order: the single-pass bars,
        # widened for recurrence (binary16 level partials) by its own rounding
        tol = max(2e-5 * abs(exact), 1e-6 * absum) if variant != "recurrence" else 2e-3 * max(abs(exact), absum * 1e-3)
        assert abs(got.value - ref.value) <= tol + 1e-6, (tag, got.value, ref.value)
