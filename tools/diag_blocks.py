import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import paper_2001_05585_b200 as T, oracle as O
for lgn in (26, 28, 30):
    n = 1 << lgn
    x = T.generate("uniform", 0, n)
    h = x.view(torch.int16).cpu().numpy().view(np.uint16)
    for (R, B) in ((1, 1024), (4, 128)):
        _, rb = O.single_pass(h, threads=16, want_blocks=True, m=16, R=R, B=B)
        for eng in (T.Engine.mma_sync_async, T.Engine.mma_sync, T.Engine.mma_sync_regs, T.Engine.tcgen05):
            gb = T.block_results(x, T.ReductionConfig(m=16, R=R, B=B, engine=eng)).cpu().numpy()
            d = gb.view(np.uint32) != rb.view(np.uint32)
            idx = np.nonzero(d)[0]
            print(lgn, R, B, eng.name, gb.size, rb.size, int(d.sum()), idx[:5].tolist(), (gb[idx[:3]].tolist(), rb[idx[:3]].tolist()), flush=True)
