#!/usr/bin/env python3
"""BASELINE configs[2] (B x R sweep at n=2^28 vs warp-shuffle and CUB) and configs[3]
(precision study, n = 2^26 .. 2^30, uniform and normal) on one B200.

    python tools/sweep.py [--sweep] [--precision] [--out gpurun_out/sweep.json]

Every point: CUDA-event time of the single_pass call (median over reps of the mean of 5
back-to-back calls, inputs > L2),
Gelem/s, GB/s and fraction of the measured HBM copy bandwidth; precision points add the
relative error against the exact sum of the binary16 inputs (device fixed-point sum) and
against the reference single_pass value (tests/golden/oracle_large.json, produced by the
pinned oracle from the reference algorithm).  --reference-csv runs the reference's own sweeps
(sweep_br, sweep_split, error_curve; harness.hpp:136-206) through the mirrored harness
(paper_2001_05585_b200/harness.py) and writes them in the csv.hpp:14-48 schema with two
wall-clock columns appended.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--precision", action="store_true")
    ap.add_argument("--variants", action="store_true")
    ap.add_argument("--reference-csv", action="store_true",
                    help="the reference's sweep_br / sweep_split / error_curve in its csv.hpp schema")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    args = ap.parse_args()
    if not (args.sweep or args.precision or args.variants or args.reference_csv):
        args.sweep = args.precision = args.variants = args.reference_csv = True

    import torch

    import paper_2001_05585_b200 as T
    from paper_2001_05585_b200 import _capi

    lib = _capi.load()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    sp = C.c_void_p(stream.cuda_stream)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    res = torch.zeros(2, dtype=torch.float32, device=dev)
    ovf = torch.zeros(1, dtype=torch.int32, device=dev)
    rp, op = C.c_void_p(res.data_ptr()), C.c_void_p(ovf.data_ptr())

    def time_fn(fn, reps):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(reps):
            # 5 back-to-back calls per sample: device throughput, host call overhead hidden
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(5):
                fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b) / 5)
        return statistics.median(ts), min(ts)

    out = {"peak_hbm_gbs": peak, "device": torch.cuda.get_device_name(0)}

    if args.sweep:
        n = 1 << 28
        x = T.generate("uniform", 0, n, device=dev)
        xp = C.c_void_p(x.data_ptr())
        pts = []
        for engine in (T.Engine.mma_sync_async, T.Engine.tcgen05, T.Engine.mma_sync, T.Engine.mma_sync_regs):
            for B in (32, 128, 256, 512, 1024):
                for R in (1, 2, 3, 4, 5):
                    cfg = T.ReductionConfig(m=16, R=R, B=B, engine=engine, finalize=T.Finalize.tree)
                    c = cfg.to_c()
                    med, best = time_fn(lambda: _capi.check(lib.tcr_single_pass_f16_async(xp, n, C.byref(c), rp, op, sp)),
                                        args.reps)
                    torch.cuda.synchronize()
                    val = res[0].item()
                    pts.append({"engine": engine.name, "B": B, "R": R, "ms": med, "ms_best": best,
                                "gelem_s": n / med / 1e6, "gb_s": 2 * n / med / 1e6,
                                "frac_hbm": 2 * n / med / 1e6 / peak, "value": val,
                                "launches": lib.tcr_last_launch_count()})
                    print(json.dumps(pts[-1]), flush=True)
        # fragment sides m != 16 (selector-matrix engine), the reference default m = 4 first
        mpts = []
        for (m, R, B) in ((4, 1, 128), (4, 4, 128), (2, 1, 128), (8, 1, 128), (8, 4, 128), (32, 1, 128), (64, 1, 128),
                          (128, 1, 128)):
            cfg = T.ReductionConfig(m=m, R=R, B=B, finalize=T.Finalize.tree)
            c = cfg.to_c()
            med, best = time_fn(lambda: _capi.check(lib.tcr_single_pass_f16_async(xp, n, C.byref(c), rp, op, sp)),
                                args.reps)
            torch.cuda.synchronize()
            mpts.append({"m": m, "R": R, "B": B, "ms": med, "gelem_s": n / med / 1e6, "gb_s": 2 * n / med / 1e6,
                         "frac_hbm": 2 * n / med / 1e6 / peak, "value": res[0].item()})
            print(json.dumps(mpts[-1]), flush=True)
        comps = {}
        comps["warp_shuffle_fp32"] = time_fn(lambda: _capi.check(lib.tcr_shuffle_f16_async(xp, n, rp, sp)), args.reps)[0]
        comps["cub_half_in_float_acc"] = time_fn(lambda: _capi.check(lib.tcr_cub_sum_f16_async(xp, n, 0, rp, sp)),
                                                 args.reps)[0]
        comps["cub_half_in_half_acc"] = time_fn(lambda: _capi.check(lib.tcr_cub_sum_f16_async(xp, n, 1, rp, sp)),
                                                args.reps)[0]
        comps["read_probe"] = time_fn(lambda: _capi.check(lib.tcr_read_probe_async(xp, 2 * n, sp)), args.reps)[0]
        out["sweep"] = {"n": n, "dist": "uniform s0", "points": pts, "m_points": mpts,
                        "comparators_ms": comps,
                        "comparators_gelem_s": {k: n / v / 1e6 for k, v in comps.items()}}
        best = min(pts, key=lambda p: p["ms"])
        out["sweep"]["best"] = best
        out["sweep"]["speedup_best_vs_warp_shuffle"] = comps["warp_shuffle_fp32"] / best["ms"]
        del x
        torch.cuda.empty_cache()

    if args.variants:
        # every reduce() variant (reduction.hpp:344-358) through the synchronous device call
        # (kernels + the 8-byte result read), n = 2^30 uniform s0, value checked against the exact sum
        n = 1 << 30
        x = T.generate("uniform", 0, n, device=dev)
        exact, _ = T.exact_sum(x)
        xp = C.c_void_p(x.data_ptr())
        # recurrence overflows binary16 on uniform input (its level partials grow past 65504, as
        # the paper reports): time it on normal(0,1) input too, where it does not
        xn = T.generate("normal", 1, n, device=dev)
        exact_n, _ = T.exact_sum(xn)
        xnp = C.c_void_p(xn.data_ptr())
        vpts = []
        # the north-star config, the reference's defaults (m = 4, reduction.hpp:41-44) and its
        # best-known per-variant configs (curve_config, harness.hpp:178-196), the m = 16 analogues
        for name, kw in (("single_pass", dict(m=16, R=1, B=1024)), ("single_pass", dict(m=4, R=1, B=128)),
                         ("single_pass", dict(m=4, R=4, B=128)), ("single_pass", dict(m=16, R=4, B=128)),
                         ("recurrence", dict(m=4, R=5, B=32)), ("recurrence", dict(m=16, R=5, B=32)),
                         ("recurrence", dict(m=4, R=1, B=32)),
                         ("recurrence", dict(m=4, R=5, B=32, dist="normal")),
                         ("recurrence", dict(m=16, R=5, B=32, dist="normal")),
                         ("split", dict(m=4, R=1, B=128, f=0.5)), ("split", dict(m=16, R=1, B=128, f=0.5)),
                         ("split", dict(m=16, R=1, B=1024, f=0.9)),
                         ("shuffle32", dict()), ("half_tree", dict()), ("oracle64", dict())):
            kw = dict(kw)
            dist = kw.pop("dist", "uniform")
            ptr, ex = (xnp, exact_n) if dist == "normal" else (xp, exact)
            cfg = T.ReductionConfig(variant=T.Variant[name], **kw)
            c = cfg.to_c()
            o = _capi.tcr_outcome()
            fn = lambda: _capi.check(lib.tcr_reduce_f16_device(ptr, n, C.byref(c), C.byref(o), sp))  # noqa: E731
            med, best = time_fn(fn, max(3, args.reps // 2))
            vpts.append({"variant": name, **kw, "dist": dist, "ms": med, "gelem_s": n / med / 1e6,
                         "gb_s": 2 * n / med / 1e6, "frac_hbm": 2 * n / med / 1e6 / peak, "value": o.value,
                         "overflow": bool(o.overflow), "rel_err_exact": abs(o.value - ex) / abs(ex),
                         "launches": lib.tcr_last_launch_count()})
            print(json.dumps(vpts[-1]), flush=True)
        out["variants"] = {"n": n, "dist": "uniform s0 (normal s1 where marked)", "exact": exact,
                           "exact_normal": exact_n, "points": vpts,
                           "timing": "CUDA events around 5 back-to-back synchronous tcr_reduce_f16_device calls"}
        del x, xn
        torch.cuda.empty_cache()

    if args.precision:
        gl = os.path.join(ROOT, "tests", "golden", "oracle_large.json")
        golden = {(r["dist"], r["seed"], r["n"]): r for r in json.load(open(gl))["cases"]} if os.path.exists(gl) else {}
        prec = []
        for dist, seed in (("uniform", 0), ("normal", 1), ("normal", 2), ("normal", 3)):
            for lgn in (26, 27, 28, 29, 30):
                n = 1 << lgn
                x = T.generate(dist, seed, n, device=dev)
                exact, absum = T.exact_sum(x)
                for (R, B) in ((1, 1024), (4, 128), (1, 128), (5, 32)):
                    for fin in (T.Finalize.tree, T.Finalize.ordered):
                        o = T.reduce(x, T.ReductionConfig(m=16, R=R, B=B, finalize=fin))
                        g = golden.get((dist, seed, n), {}).get("single_pass", {}).get(f"m16_R{R}_B{B}")
                        rec = {"dist": dist, "seed": seed, "n": n, "R": R, "B": B, "finalize": fin.name,
                               "value": o.value, "overflow": o.overflow, "exact": exact, "abs_sum": absum,
                               "rel_err_exact": abs(o.value - exact) / abs(exact),
                               "err_over_abs_sum": abs(o.value - exact) / absum,
                               "reference_value": g["value"] if g else None,
                               "rel_diff_reference": (abs(o.value - g["value"]) / abs(exact)) if g else None,
                               "reference_rel_err_exact": (abs(g["value"] - exact) / abs(exact)) if g else None}
                        prec.append(rec)
                        print(json.dumps(rec), flush=True)
                del x
                torch.cuda.empty_cache()
        out["precision"] = prec

    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    if args.reference_csv:
        # the reference's own sweeps (harness.hpp:136-206) through the mirrored harness: fp32 inputs,
        # reduce() + oracle64 on the B200, rows in the csv.hpp:14-48 schema (+ ms, Gelem/s of the
        # synchronous reduce call)
        from paper_2001_05585_b200 import harness as H
        du = H.Distribution(T.DistKind.uniform, 0)
        dists = [du] + [H.Distribution(T.DistKind.normal, s) for s in (1, 2, 3)]
        sizes = [1 << k for k in range(26, 31)]
        sets = {
            "sweep_br_m16": lambda: H.sweep_br(du, 1 << 28, T.Variant.single_pass, H.default_block_grid(),
                                               H.default_chain_grid(), m=16),
            "sweep_br_m4": lambda: H.sweep_br(du, 1 << 28, T.Variant.single_pass, H.default_block_grid(),
                                              H.default_chain_grid()),
            "sweep_split": lambda: H.sweep_split(du, 1 << 28, H.default_fraction_grid()),
            "error_curve": lambda: [r for d in dists for v in (T.Variant.single_pass, T.Variant.recurrence,
                                                                T.Variant.split, T.Variant.shuffle32,
                                                                T.Variant.half_tree)
                                    for r in H.error_curve(d, v, sizes)],
        }
        base = os.path.splitext(args.out)[0]
        for name, fn in sets.items():
            recs = fn()
            with open(f"{base}_{name}.csv", "w") as f:
                H.write_csv(f, recs, wall_clock=True)
            best = H.best_by_steps_per_element(recs)
            print(f"{name}: {len(recs)} rows -> {base}_{name}.csv; best by sim_steps/element: {H.csv_row(best)}",
                  flush=True)
            torch.cuda.empty_cache()

if __name__ == "__main__":
    main()
