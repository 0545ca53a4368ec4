"""Multi-GPU shard + combine for single_pass (BASELINE configs[4]).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  The global input is cut
into contiguous shards aligned to the kernel's group size (G logical blocks), so every rank's
block and group partition is a sub-partition of the single-GPU one: only the last rank can
have a ragged tail, exactly like the reference's zero padding (reduction.hpp:244-245).  Each
rank reduces its shard with the sm_100a kernel (result stays on the device), then ONE
collective combines the fp32 partials:

  combine="allreduce"  one ncclAllReduce(sum) of the 4-byte partial (the north-star design);
  combine="tree"       one all_gather of the N partials + the fixed adjacent pairwise tree
                       over rank order.  With N a power of two and equal power-of-two group
                       counts per rank this is BIT-IDENTICAL to the single-GPU tree finaliser.
"""
from __future__ import annotations

import dataclasses

from .reduction import ReductionConfig, ReductionOutcome, counters


@dataclasses.dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    first: int      # first global element of this shard
    count: int      # elements in this shard (may be 0 for trailing ranks of tiny inputs)


def group_elems(cfg: ReductionConfig) -> int:
    """Elements per kernel group (G logical blocks): the shard alignment (tcr_group_elems)."""
    import ctypes as C
    from . import _capi
    c = cfg.to_c()
    ge = _capi.load().tcr_group_elems(C.byref(c))
    if ge == 0:
        cfg.validate()
    return ge


def shard(n_total: int, rank: int, world: int, cfg: ReductionConfig) -> Shard:
    """Contiguous shard of rank `rank`, boundaries on multiples of group_elems(cfg)."""
    if n_total <= 0:
        raise ValueError("input must be non-empty")
    if not 0 <= rank < world:
        raise ValueError("bad rank")
    ge = group_elems(cfg)
    groups = -(-n_total // ge)
    per = -(-groups // world)
    g0, g1 = min(groups, rank * per), min(groups, (rank + 1) * per)
    first = g0 * ge
    last = min(n_total, g1 * ge)
    return Shard(rank, world, first, max(0, last - first))


def tree_combine(parts: list[float]) -> float:
    """Adjacent pairwise tree over `parts` in rank order, zero padded to a power of two
    (the same order the kernel's finaliser uses over group partials)."""
    import numpy as np
    v = [np.float32(p) for p in parts]
    P = 1
    while P < len(v):
        P <<= 1
    v += [np.float32(0.0)] * (P - len(v))
    while len(v) > 1:
        v = [np.float32(v[2 * i] + v[2 * i + 1]) for i in range(len(v) // 2)]
    return float(v[0])


def combine(partial, overflow, group=None, how: str = "allreduce"):
    """Combine per-rank fp32 partials (1-element tensors on any device) across the process group
    with ONE collective.  Returns (value, overflow) as Python scalars.

    The overflow flag needs no collective of its own: a rank's flag is set iff its partial is
    non-finite (every overflow note of reduction.hpp:78-81 comes from a non-finite binary16 value
    -- an input or a C_R column sum -- whose chunk result is then non-finite, and a non-finite
    value stays non-finite through the fp32 tree; finite binary16 data cannot overflow an fp32
    sum of fewer than 2^100 elements), so the combined flag is "the combined value is not finite"."""
    import math

    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(partial.item()), bool(int(overflow.item()))
    if how == "allreduce":
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
        value = float(partial.item())
        return value, not math.isfinite(value)
    if how == "tree":
        world = dist.get_world_size(group)
        out = [torch.zeros_like(partial) for _ in range(world)]
        dist.all_gather(out, partial, group=group)
        parts = [float(t.item()) for t in out]
        return tree_combine(parts), not all(math.isfinite(p) for p in parts)
    raise ValueError(f"unknown combine {how!r}")


def reduce_sharded(x_local, n_total: int, cfg: ReductionConfig, group=None, how: str = "allreduce",
                   partial_fn=None) -> ReductionOutcome:
    """single_pass over a sharded input: x_local is this rank's shard (CUDA float16 tensor,
    from shard()).  partial_fn(x_local, cfg) -> (partial, overflow) tensors; defaults to the
    sm_100a kernel via tcr_single_pass_f16_async (override only in host-logic unit tests)."""
    import torch
    if partial_fn is None:
        from .reduction import single_pass_async
        res = torch.zeros(1, dtype=torch.float32, device=x_local.device)
        ovf = torch.zeros(1, dtype=torch.int32, device=x_local.device)
        if x_local.numel() > 0:
            single_pass_async(x_local, cfg, res, ovf)
        partial, overflow = res, ovf
    else:
        partial, overflow = partial_fn(x_local, cfg)
    value, ov = combine(partial, overflow, group, how)
    out = counters(n_total, cfg)
    out.value = value
    out.overflow = ov
    return out
