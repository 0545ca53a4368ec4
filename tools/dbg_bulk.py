import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2001_05585_b200 as T
sys.path.insert(0, "oracle"); import oracle as O
x = O.generate("integers", 0, 1 << 20)
xd = torch.from_numpy(x).cuda().half()
for R, B in [(3, 32), (3, 64), (5, 32), (3, 128), (1, 32), (2, 32)]:
    a = T.block_results(xd, T.ReductionConfig(m=16, R=R, B=B, engine=T.Engine.mma_sync_regs)).cpu().numpy()
    b = T.block_results(xd, T.ReductionConfig(m=16, R=R, B=B, engine=T.Engine.mma_sync)).cpu().numpy()
    bad = np.nonzero(a != b)[0]
    g = T.sharded.group_elems(T.ReductionConfig(m=16, R=R, B=B)) // (R * 256 * (B // 32))
    print(R, B, "G", g, "nblocks", len(a), "mismatch", len(bad), bad[:20], bad[-5:] if len(bad) else "")
