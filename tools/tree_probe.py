import sys, ctypes as C
sys.path.insert(0, '.')
import torch
import paper_2001_05585_b200 as T
from paper_2001_05585_b200 import _capi
lib = _capi.load()
n = 1 << 30
x = T.generate("uniform", 0, n, device="cuda")
for v in ("shuffle32", "half_tree"):
    o = T.reduce(x, T.ReductionConfig(variant=T.Variant[v]))
    print(v, o.value)
