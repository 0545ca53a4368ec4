"""Python mirror of the reference's sweep harness and CSV schema over the device path.

    Distribution, generate          harness.hpp:20-80     (inputs generated on the device, bit-exact)
    error_percent                   harness.hpp:83-87
    SweepRecord, run_point          harness.hpp:89-117    (reduce() and oracle64 run on the B200)
    default_*_grid                  harness.hpp:119-136
    sweep_br, sweep_split           harness.hpp:138-175
    curve_config, error_curve       harness.hpp:177-206
    best_by_steps_per_element       harness.hpp:208-217
    CSV_HEADER, csv_row, write_csv  csv.hpp:14-53

Same names, argument meaning and error behaviour (std::invalid_argument -> ValueError).  A record
is a deterministic function of (distribution, seed, n, config), as in the reference; the one
addition is ``SweepRecord.ms`` (device time of the reduce call), which ``write_csv`` appends as
wall-clock columns only when asked, so the default output is the reference's fixed schema.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

from .reduction import DistKind, ReductionConfig, ReductionOutcome, Variant, reduce, variant_name
from .reduction import generate as _device_generate

CSV_HEADER = "variant,n,m,R,B,f,seed,dist,value,error_pct,overflow,sim_steps,mma_count,atomic_count"  # csv.hpp:14-15
WALL_CLOCK_COLUMNS = "ms,gelem_s"


@dataclasses.dataclass
class Distribution:                       # harness.hpp:22-45
    kind: DistKind = DistKind.uniform
    seed: int = 0
    lo: int = 0                           # integers(lo, hi), inclusive
    hi: int = 9
    c: float = 1.0                        # constant(c)

    def name(self) -> str:
        k = DistKind(self.kind)
        if k == DistKind.integers:
            return f"integers:{self.lo}:{self.hi}"
        if k == DistKind.constant:
            return "constant:" + _c_format("%g", self.c)
        return k.name


def generate(dist: Distribution, n: int, device="cuda"):
    """harness.hpp:47-80: the reference's generator, as a float32 CUDA tensor (bit-exact)."""
    if n < 1:
        raise ValueError("generate requires n >= 1")
    if DistKind(dist.kind) == DistKind.integers and dist.hi < dist.lo:
        raise ValueError("integers: hi < lo")
    return _device_generate(int(dist.kind), dist.seed, n, device=device, dtype="float32", lo=dist.lo, hi=dist.hi,
                            c=dist.c)


def error_percent(value: float, reference: float) -> Optional[float]:   # harness.hpp:83-87
    if reference == 0.0:
        return None
    return 100.0 * abs(value - reference) / abs(reference)


@dataclasses.dataclass
class SweepRecord:                        # harness.hpp:89-100
    config: ReductionConfig = dataclasses.field(default_factory=ReductionConfig)
    n: int = 0
    seed: int = 0
    dist: str = ""
    value: float = 0.0
    error_pct: Optional[float] = None
    overflow: bool = False
    sim_steps: int = 0
    mma_count: int = 0
    atomic_count: int = 0
    ms: Optional[float] = None            # B200 addition: device time of the reduce call


def _timed_reduce(x, cfg: ReductionConfig) -> tuple[ReductionOutcome, float]:
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream(x.device)
    a.record(s)
    out = reduce(x, cfg)                  # synchronous: ends with the 8-byte result read
    b.record(s)
    b.synchronize()
    return out, a.elapsed_time(b)


def run_point(dist: Distribution, n: int, cfg: ReductionConfig) -> SweepRecord:
    """harness.hpp:103-117: generate, reduce(std::span<const float>), error against oracle64 of
    the same float32 input (skipped on overflow)."""
    x = generate(dist, n)
    out, ms = _timed_reduce(x, cfg)
    rec = SweepRecord(config=cfg, n=n, seed=dist.seed, dist=dist.name(), value=out.value, overflow=out.overflow,
                      sim_steps=out.sim_steps, mma_count=out.mma_count, atomic_count=out.atomic_count, ms=ms)
    if not out.overflow:
        ref = reduce(x, ReductionConfig(variant=Variant.oracle64)).value
        rec.error_pct = error_percent(out.value, ref)
    return rec


def default_block_grid() -> list[int]:    # harness.hpp:119-122
    return [32, 64, 128, 256, 512, 1024]


def default_chain_grid() -> list[int]:    # harness.hpp:124-127
    return [1, 2, 3, 4, 5, 6, 7, 8]


def default_fraction_grid() -> list[float]:   # harness.hpp:129-133
    return [i / 10.0 for i in range(11)]


def sweep_br(dist: Distribution, n: int, variant: Variant, block_grid, chain_grid, m: int = 4) -> list[SweepRecord]:
    """harness.hpp:136-157: one record per (B, R), B outer, R inner."""
    if not block_grid or not chain_grid:
        raise ValueError("sweep grids must be non-empty")
    return [run_point(dist, n, ReductionConfig(variant=Variant(variant), m=m, R=chain, B=blk))
            for blk in block_grid for chain in chain_grid]


def sweep_split(dist: Distribution, n: int, fraction_grid, block: int = 128, m: int = 4) -> list[SweepRecord]:
    """harness.hpp:159-175: one record per split fraction."""
    if not fraction_grid:
        raise ValueError("sweep grids must be non-empty")
    return [run_point(dist, n, ReductionConfig(variant=Variant.split, m=m, R=1, B=block, f=frac))
            for frac in fraction_grid]


def curve_config(variant: Variant) -> ReductionConfig:   # harness.hpp:177-196
    v = Variant(variant)
    if v == Variant.single_pass:
        return ReductionConfig(variant=v, B=128, R=4)
    if v == Variant.recurrence:
        return ReductionConfig(variant=v, B=32, R=5)
    return ReductionConfig(variant=v, B=128, R=1)


def error_curve(dist: Distribution, variant: Variant, n_grid) -> list[SweepRecord]:   # harness.hpp:198-206
    cfg = curve_config(variant)
    return [run_point(dist, n, cfg) for n in n_grid]


def best_by_steps_per_element(records) -> SweepRecord:   # harness.hpp:208-217
    if not records:
        raise ValueError("no records")
    best = records[0]
    for rec in records:
        if rec.sim_steps / rec.n < best.sim_steps / best.n:
            best = rec
    return best


# ------------------------------------------------------------------------------------- csv.hpp

def _c_format(spec: str, v: float) -> str:
    """printf(spec, v) as glibc prints it: Python's %-formatting is correctly rounded like glibc's;
    only the NaN sign differs (glibc prints "-nan" for a NaN with the sign bit set)."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    return spec % v


def fmt_double(v: float) -> str:          # csv.hpp:19-25
    return _c_format("%.9g", float(v))


def csv_row(rec: SweepRecord, wall_clock: bool = False) -> str:   # csv.hpp:27-48
    c = rec.config
    row = ",".join([variant_name(c.variant), str(rec.n), str(c.m), str(c.R), str(c.B), fmt_double(c.f),
                    str(rec.seed), rec.dist, fmt_double(rec.value),
                    fmt_double(rec.error_pct) if rec.error_pct is not None else "nan",
                    "true" if rec.overflow else "false", str(rec.sim_steps), str(rec.mma_count),
                    str(rec.atomic_count)])
    if wall_clock:
        ms = rec.ms
        row += "," + (fmt_double(ms) if ms is not None else "nan")
        row += "," + (fmt_double(rec.n / (ms * 1e6)) if ms else "nan")
    return row


def write_csv(os_, records, wall_clock: bool = False) -> None:   # csv.hpp:50-53
    """Header + one row per record.  wall_clock=True appends the B200 device-time columns
    (ms, Gelem/s) after the reference's fixed 14."""
    os_.write(CSV_HEADER + ("," + WALL_CLOCK_COLUMNS if wall_clock else "") + "\n")
    for rec in records:
        os_.write(csv_row(rec, wall_clock) + "\n")
