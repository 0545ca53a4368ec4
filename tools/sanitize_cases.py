#!/usr/bin/env python3
"""Small reductions over every engine / fragment side / variant, for compute-sanitizer
(memcheck, racecheck, synccheck, initcheck):
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
Each case is checked against the oracle so a sanitizer run is also a parity run."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402  (checker)
import paper_2001_05585_b200 as T  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    n = (1 << 18) + 4097                       # several groups plus a ragged tail
    h = O.generate("integers", 3, n).astype(np.float16).view(np.uint16)
    x = torch.from_numpy(h.view(np.int16).copy()).to(dev).view(torch.float16)
    exact = float(O.generate("integers", 3, n).astype(np.float64).sum())
    cases = []
    for eng in (T.Engine.mma_sync_async, T.Engine.mma_sync, T.Engine.mma_sync_regs, T.Engine.tcgen05):
        for R, B in ((1, 1024), (3, 96), (8, 32)):
            cases.append(("single_pass", dict(m=16, R=R, B=B, engine=eng)))
    for m, R, B in ((2, 1, 128), (2, 3, 64), (4, 1, 128), (4, 1, 64), (4, 1, 1024), (4, 5, 32), (8, 1, 128), (8, 3, 32), (32, 1, 128),
                    (128, 1, 32), (256, 1, 32), (1024, 1, 32), (4096, 1, 32)):
        cases.append(("single_pass", dict(m=m, R=R, B=B)))
    for fin in (T.Finalize.ordered, T.Finalize.atomic):
        cases.append(("single_pass", dict(m=16, R=1, B=1024, finalize=fin)))
        cases.append(("single_pass", dict(m=4, R=1, B=128, finalize=fin)))
    for v in ("recurrence", "split", "shuffle32", "half_tree", "oracle64"):
        cases.append((v, dict(m=16, R=5, B=32)))
    bad = 0
    for v, kw in cases:
        cfg = T.ReductionConfig(variant=T.Variant[v], **kw)
        o = T.reduce(x, cfg)
        # half_tree / recurrence store partials through binary16 and overflow on these inputs
        ok = o.value == exact or v in ("half_tree", "recurrence")
        bad += 0 if ok else 1
        print(f"{'ok ' if ok else 'BAD'} {v} {kw}: {o.value}", flush=True)
    xf = x.float()
    o = T.reduce(xf, T.ReductionConfig(m=16, R=1, B=1024))
    print("ok " if o.value == exact else "BAD", "fp32 device", o.value, flush=True)
    o = T.reduce(h.view(np.float16), T.ReductionConfig(m=16, R=1, B=1024))
    print("ok " if o.value == exact else "BAD", "binary16 host", o.value, flush=True)
    torch.cuda.synchronize()
    print("cases", len(cases) + 2, "mismatches", bad)


if __name__ == "__main__":
    main()
