import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, torch
import oracle as O
import paper_2001_05585_b200 as T
n = (1 << 20) + 4097
h = O.generate("integers", 3, n).astype(np.float16).view(np.uint16)
x = torch.from_numpy(h.view(np.int16).copy()).cuda().view(torch.float16)
exact = float(O.generate("integers", 3, n).astype(np.float64).sum())
for R, B in ((1, 1024), (3, 96), (8, 32), (2, 256)):
    for fin in (T.Finalize.tree, T.Finalize.ordered):
        o = T.reduce(x, T.ReductionConfig(m=16, R=R, B=B, engine=T.Engine.mma_sync, finalize=fin))
        print(R, B, fin.name, o.value, exact, T.reduction.last_engine().name, flush=True)
        assert o.value == exact
