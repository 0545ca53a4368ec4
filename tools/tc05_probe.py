"""Quick tcgen05-engine probe (run under `timeout`): small cases vs the mma.sync engine."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2001_05585_b200 as T
ok = True
for (n, R, B, dist) in [(1 << 16, 1, 1024, "integers"), (1 << 20, 1, 1024, "uniform"), ((1 << 20) + 999, 4, 128, "normal"),
                        (1 << 22, 3, 96, "uniform"), (1 << 22, 5, 32, "normal"), (1 << 24, 2, 256, "uniform")]:
    x = T.generate(dist, 1, n)
    a = T.reduce(x, T.ReductionConfig(m=16, R=R, B=B, engine=T.Engine.mma_sync))
    torch.cuda.synchronize()
    b = T.reduce(x, T.ReductionConfig(m=16, R=R, B=B, engine=T.Engine.tcgen05))
    torch.cuda.synchronize()
    print(n, R, B, dist, "mma_sync", a.value, "tcgen05", b.value, "launches", T.reduction.last_launch_count(), flush=True)
    ok &= abs(a.value - b.value) <= 1e-6 * abs(a.value) + 1e-3
print("TC05 PROBE", "OK" if ok else "MISMATCH")
