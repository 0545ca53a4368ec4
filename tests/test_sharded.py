"""Multi-process (gloo, world_size 2, CPU) tests of the shard + combine host logic
(paper_2001_05585_b200/sharded.py).  The per-rank partial is emulated from the oracle's block
results with the kernel's own group/tree order (the GPU is not available here); on the B200
the same reduce_sharded() call runs the sm_100a kernel and NCCL instead."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2001_05585_b200 as T
from paper_2001_05585_b200 import sharded as S


def adjacent_tree(vals):
    v = [np.float32(x) for x in vals]
    P = 1
    while P < len(v):
        P <<= 1
    v += [np.float32(0)] * (P - len(v))
    while len(v) > 1:
        v = [np.float32(v[2 * i] + v[2 * i + 1]) for i in range(len(v) // 2)]
    return np.float32(v[0])


def emulated_tree_value(oracle, h, cfg):
    """What the kernel's TREE finaliser returns for input h: block results (reference
    semantics), adjacent tree inside each group of G blocks, adjacent tree over groups."""
    _, blocks = oracle.single_pass(h, threads=4, want_blocks=True, m=cfg.m, R=cfg.R, B=cfg.B)
    G = S.group_elems(cfg) // (cfg.R * cfg.m * cfg.m * (cfg.B // 32))
    groups = [adjacent_tree(blocks[i:i + G].tolist() + [0.0] * (G - len(blocks[i:i + G])))
              for i in range(0, len(blocks), G)]
    return float(adjacent_tree(groups))


def test_shard_plan_properties():
    for R, B in ((1, 1024), (4, 128), (5, 96), (3, 32)):
        cfg = T.ReductionConfig(m=16, R=R, B=B)
        ge = S.group_elems(cfg)
        for n in (1, 1000, ge, ge + 1, 8 * ge, (1 << 30) + 12345):
            for world in (1, 2, 4, 8):
                shards = [S.shard(n, r, world, cfg) for r in range(world)]
                assert shards[0].first == 0
                assert sum(s.count for s in shards) == n
                for a, b in zip(shards, shards[1:]):
                    assert b.first == a.first + a.count or b.count == 0
                nonempty = [s for s in shards if s.count]
                for s in nonempty[:-1]:
                    assert s.count % ge == 0 and s.first % ge == 0  # only the last shard may be ragged
    with pytest.raises(ValueError):
        S.shard(0, 0, 1, T.ReductionConfig(m=16))


def test_tree_combine_matches_single_tree():
    rng = np.random.default_rng(3)
    vals = rng.random(8).astype(np.float32)
    assert S.tree_combine(vals.tolist()) == float(adjacent_tree(vals.tolist()))
    assert S.tree_combine([1.0]) == 1.0
    assert S.tree_combine([1.0, 2.0, 3.0]) == 6.0


def _worker(rank, world, port, n, how, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle as O
    cfg = T.ReductionConfig(m=16, R=1, B=1024)
    sh = S.shard(n, rank, world, cfg)
    h = O.generate_f16("uniform", 0, sh.count, first=sh.first)

    def partial_fn(x, c):
        v = emulated_tree_value(O, x, c)
        return torch.tensor([v], dtype=torch.float32), torch.tensor([0], dtype=torch.int32)

    out = S.reduce_sharded(h, n, cfg, how=how, partial_fn=partial_fn)

    def overflow_fn(x, c):  # rank 1 overflowed: its kernel partial is non-finite with the flag set
        v = float("inf") if rank == 1 else 1.0
        return torch.tensor([v], dtype=torch.float32), torch.tensor([int(rank == 1)], dtype=torch.int32)

    def mixed_fn(x, c):    # +inf on rank 0, -inf on rank 1: the combined value is NaN, still flagged
        v = float("inf") if rank == 0 else float("-inf")
        return torch.tensor([v], dtype=torch.float32), torch.tensor([1], dtype=torch.int32)

    out2 = S.reduce_sharded(h, n, cfg, how=how, partial_fn=overflow_fn)
    out3 = S.reduce_sharded(h, n, cfg, how=how, partial_fn=mixed_fn)
    out_q.put((rank, out.value, out.overflow, out.atomic_count, out.mma_count, out2.overflow and out3.overflow))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("how", ["tree", "allreduce"])
def test_two_rank_gloo_combine(oracle, how):
    n = 4 * 65536 * 2  # 4 groups per rank at m16 R1 B1024
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + (7 if how == "tree" else 0)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, how, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = emulated_tree_value(oracle, oracle.generate_f16("uniform", 0, n), T.ReductionConfig(m=16, R=1, B=1024))
    exact, _ = oracle.exact_sum_f16(oracle.generate_f16("uniform", 0, n))
    ref_counts = T.counters(n, T.ReductionConfig(m=16, R=1, B=1024))
    for rank, value, ovf, atomics, mmas, ovf2 in res:
        assert not ovf and ovf2  # overflow on any rank is seen by all ranks (one collective)
        assert atomics == ref_counts.atomic_count and mmas == ref_counts.mma_count
        if how == "tree":
            assert value == single  # bit-identical to the single-GPU tree finaliser
        else:
            # one fp32 rounding away from the single-GPU tree; method error vs exact as the reference
            assert abs(value - single) <= 2.0 ** -22 * abs(single)
            assert abs(value - exact) / exact < 1e-5
    assert res[0][1] == res[1][1]
