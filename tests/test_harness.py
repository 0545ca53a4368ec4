"""The reference's sweep harness and CSV schema (harness.hpp, csv.hpp) mirrored over the device
path (paper_2001_05585_b200/harness.py).

CPU: csv_row / the header against the reference's own csv_row (csv.hpp:19-48, compiled as-is in
oracle/_ref) on records with identical fields -- every formatting branch (%.9g, nan error,
true/false, inf / -inf / nan / -nan / -0 / subnormal / huge values, every variant).
GPU: run_point / sweep_br / sweep_split / error_curve on the B200 against the reference's
run_point on the CPU -- byte-identical rows on exact inputs for every variant and on uniform
inputs for single_pass (the ORDERED default combine and the bit-exact oracle64), every non-float
column identical and the value within the precision bars elsewhere."""
import io
import math
import random

import numpy as np
import pytest

import paper_2001_05585_b200 as T
from paper_2001_05585_b200 import harness as H

from conftest import has_gpu

VARIANT_NAMES = ["oracle64", "shuffle32", "half_tree", "recurrence", "single_pass", "split"]


def _ref_or_skip(oracle):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")


def test_csv_header_is_the_reference_schema(oracle):
    _ref_or_skip(oracle)
    assert H.CSV_HEADER == oracle.ref_csv_header()
    buf = io.StringIO()
    H.write_csv(buf, [])
    assert buf.getvalue() == oracle.ref_csv_header() + "\n"
    buf = io.StringIO()
    H.write_csv(buf, [], wall_clock=True)
    assert buf.getvalue().startswith(oracle.ref_csv_header() + ",")


def _special_values(rng):
    vals = [0.0, -0.0, 1.0, -1.0, 0.5, 1e-45, 1.401298464324817e-45, 5e-324, 2.2250738585072014e-308, 65504.0,
            65520.0, 3.4028234663852886e38, 1e300, -1e-300, math.inf, -math.inf, math.nan, -math.nan, 536864032.0,
            134221184.0, 0.1, 1 / 3, 2 / 3, 123456789.0, 1234567890123.0, 9.999999995e-5, 1e-4, 1e16, 1e17,
            99999999.95, 0.000123456789012]
    vals += [rng.uniform(-1e9, 1e9) for _ in range(40)]
    vals += [float(np.float32(rng.gauss(0, 1e4))) for _ in range(40)]
    vals += [math.ldexp(rng.random(), rng.randint(-1070, 1020)) for _ in range(40)]
    return vals


def test_csv_row_matches_reference_formatting(oracle):
    _ref_or_skip(oracle)
    rng = random.Random(7)
    vals = _special_values(rng)
    errs = [None, 0.0, 1e-7, 3.0993e-4, 100.0, 12.5, math.inf, 4.411e-6] + [rng.random() * 10 ** rng.randint(-9, 3)
                                                                           for _ in range(20)]
    fs = [0.0, 0.1, 0.5, 0.3, 1.0, 0.7000000000000001]
    dists = ["uniform", "normal", "integers:0:9", "integers:-5:5", "constant:1", "constant:0.1"]
    n_rows = 0
    for i, v in enumerate(vals):
        variant = i % 6
        cfg = dict(variant=VARIANT_NAMES[variant], m=[2, 4, 8, 16, 1024][i % 5], R=1 + i % 8,
                   B=[32, 128, 1024][i % 3], f=fs[i % len(fs)])
        for err in (errs[i % len(errs)], None):
            rec = H.SweepRecord(config=T.ReductionConfig(variant=T.Variant(variant), m=cfg["m"], R=cfg["R"],
                                                         B=cfg["B"], f=cfg["f"]),
                                n=(1 << (i % 34)) + i, seed=i * 7919, dist=dists[i % len(dists)], value=v,
                                error_pct=err, overflow=bool(i & 1), sim_steps=i * 3 + 1, mma_count=i << 20,
                                atomic_count=(1 << 40) + i)
            ref = oracle.ref_csv_row(rec.n, rec.seed, rec.dist, v, err, rec.overflow, rec.sim_steps, rec.mma_count,
                                     rec.atomic_count, **cfg)
            assert H.csv_row(rec) == ref, (v, err)
            n_rows += 1
    assert n_rows == 2 * len(vals)


def test_harness_host_logic_matches_reference():
    # harness.hpp:119-133 grids, :177-196 curve_config, :83-87 error_percent, :22-45 names
    assert H.default_block_grid() == [32, 64, 128, 256, 512, 1024]
    assert H.default_chain_grid() == list(range(1, 9))
    assert H.default_fraction_grid() == [i / 10.0 for i in range(11)]
    sp = H.curve_config(T.Variant.single_pass)
    assert (sp.B, sp.R, sp.m) == (128, 4, 4)
    rc = H.curve_config(T.Variant.recurrence)
    assert (rc.B, rc.R) == (32, 5)
    for v in (T.Variant.oracle64, T.Variant.shuffle32, T.Variant.half_tree, T.Variant.split):
        c = H.curve_config(v)
        assert (c.B, c.R, c.variant) == (128, 1, v)
    assert H.error_percent(1.0, 0.0) is None
    assert H.error_percent(99.0, 100.0) == 1.0
    assert H.Distribution(T.DistKind.integers, 0, -3, 7).name() == "integers:-3:7"
    assert H.Distribution(T.DistKind.constant, c=0.25).name() == "constant:0.25"
    assert H.Distribution(T.DistKind.normal).name() == "normal"
    with pytest.raises(ValueError):
        H.sweep_br(H.Distribution(), 16, T.Variant.single_pass, [], [1])
    with pytest.raises(ValueError):
        H.sweep_split(H.Distribution(), 16, [])
    with pytest.raises(ValueError):
        H.best_by_steps_per_element([])
    recs = [H.SweepRecord(n=100, sim_steps=50), H.SweepRecord(n=200, sim_steps=60), H.SweepRecord(n=300, sim_steps=90)]
    assert H.best_by_steps_per_element(recs) is recs[1]   # ties keep grid order (0.3 == 0.3: first)


# ------------------------------------------------------------------------------------------- GPU

def _ref_row(oracle, dist: H.Distribution, n, cfg: T.ReductionConfig):
    return oracle.ref_run_point_csv(T.DistKind(dist.kind).name, dist.seed, n, dist.lo, dist.hi, dist.c,
                                    variant=int(cfg.variant), m=cfg.m, R=cfg.R, B=cfg.B, f=cfg.f)


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a GPU")
@pytest.mark.parametrize("variant", list(T.Variant))
@pytest.mark.parametrize("dist", [H.Distribution(T.DistKind.integers, 0, 0, 9), H.Distribution(T.DistKind.integers, 3, -7, 7),
                                  H.Distribution(T.DistKind.constant, 0, c=1.0)])
def test_run_point_rows_byte_identical_on_exact_inputs(oracle, variant, dist):
    """Integer and constant inputs: every variant's sums are exact (or overflow identically), so
    the whole csv.hpp row -- value and oracle64 error included -- equals the reference's."""
    _ref_or_skip(oracle)
    for n, m, R, B in [(1000, 4, 1, 128), (1 << 14, 16, 4, 128), (12345, 8, 2, 64), (1 << 16, 2, 3, 32)]:
        cfg = T.ReductionConfig(variant=variant, m=m, R=R, B=B)
        got = H.csv_row(H.run_point(dist, n, cfg))
        assert got == _ref_row(oracle, dist, n, cfg)


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a GPU")
def test_sweeps_match_reference_rows(oracle):
    """sweep_br (B outer, R inner), sweep_split and error_curve on uniform / normal inputs: every
    column but value and error_pct identical to the reference's run_point rows; the value within
    the precision bars of tests/test_gpu_parity.py; best_by_steps_per_element picks the same row."""
    _ref_or_skip(oracle)
    cases = []
    du, dn = H.Distribution(T.DistKind.uniform, 0), H.Distribution(T.DistKind.normal, 1)
    cases += [(du, r) for r in H.sweep_br(du, 1 << 15, T.Variant.single_pass, [32, 128, 1024], [1, 2, 5])]
    cases += [(dn, r) for r in H.sweep_br(dn, 40000, T.Variant.single_pass, [64, 256], [1, 4], m=16)]
    cases += [(du, r) for r in H.sweep_split(du, 1 << 14, [0.0, 0.3, 0.5, 1.0])]
    cases += [(dn, r) for r in H.error_curve(dn, T.Variant.single_pass, [1000, 1 << 14, 1 << 16])]
    refs = []
    for dist, rec in cases:
        ref = _ref_row(oracle, dist, rec.n, rec.config).split(",")
        got = H.csv_row(rec).split(",")
        refs.append(ref)
        assert got[:8] == ref[:8] and got[10:] == ref[10:], (got, ref)
        rv, gv = float(ref[8]), float(got[8])
        tol = 1e-5 * max(1.0, abs(rv)) if dist.kind == T.DistKind.uniform else 1e-3 * max(1.0, math.sqrt(rec.n))
        assert abs(gv - rv) <= tol, (got, ref)
    br = [rec for _, rec in cases[:9]]
    best = H.best_by_steps_per_element(br)
    ref_steps = [int(r[11]) / int(r[1]) for r in refs[:9]]
    assert br.index(best) == ref_steps.index(min(ref_steps))
    buf = io.StringIO()
    H.write_csv(buf, br, wall_clock=True)
    lines = buf.getvalue().splitlines()
    assert len(lines) == 10 and lines[0].startswith(H.CSV_HEADER + ",ms,gelem_s")
    assert all(len(line.split(",")) == 16 for line in lines[1:])


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a GPU")
@pytest.mark.parametrize("m,R,B", [(16, 1, 1024), (4, 1, 128), (4, 4, 128), (16, 4, 128), (8, 2, 64)])
def test_run_point_rows_byte_identical_uniform(oracle, m, R, B):
    """Uniform inputs (the paper's figures): with the drop-in default ORDERED combine and the
    bit-exact oracle64, the whole csv.hpp row -- value and error_pct included -- equals the
    reference's wherever the device block results are the reference's (100 % on uniform data)."""
    _ref_or_skip(oracle)
    du = H.Distribution(T.DistKind.uniform, 0)
    for n in (1 << 14, 100003, 1 << 18):
        cfg = T.ReductionConfig(m=m, R=R, B=B)
        assert H.csv_row(H.run_point(du, n, cfg)) == _ref_row(oracle, du, n, cfg)
