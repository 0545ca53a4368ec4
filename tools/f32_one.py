import sys, ctypes as C
sys.path.insert(0, '.')
import torch
import paper_2001_05585_b200 as T
from paper_2001_05585_b200 import _capi
lib = _capi.load()
dev = torch.device('cuda', 0); st = torch.cuda.current_stream(dev)
n = 1 << 28
xf = T.generate('uniform', 0, n, device=dev, dtype='float32')
res = torch.zeros(2, dtype=torch.float32, device=dev); ovf = torch.zeros(1, dtype=torch.int32, device=dev)
cfg = T.ReductionConfig(m=16, R=1, B=1024).to_c()
for _ in range(3):
    _capi.check(lib.tcr_single_pass_f32_async(C.c_void_p(xf.data_ptr()), n, C.byref(cfg), C.c_void_p(res.data_ptr()), C.c_void_p(ovf.data_ptr()), C.c_void_p(st.cuda_stream)))
torch.cuda.synchronize()
