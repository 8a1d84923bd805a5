"""One fused BatchNorm forward + backward through the C-ABI (ncu target).
usage: python tools/bn_one.py P C [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_12780_b200 import _native as N

lib = N.load()
P, C = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
bf = torch.bfloat16
z, dy = torch.randn(P, C, device="cuda").to(bf), torch.randn(P, C, device="cuda").to(bf)
y, dz = torch.empty_like(z), torch.empty_like(z)
g, b = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
mean, rstd, dg, db = (torch.empty(C, device="cuda") for _ in range(4))
ws = torch.empty(lib.ppll_batchnorm_ws_floats(P, C), device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    lib.ppll_batchnorm_fwd(P, C, z.data_ptr(), g.data_ptr(), b.data_ptr(), None, 1, y.data_ptr(),
                           mean.data_ptr(), rstd.data_ptr(), ws.data_ptr(), ws.numel(), N.BF16, s)
    lib.ppll_batchnorm_bwd(P, C, dy.data_ptr(), z.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                           g.data_ptr(), dg.data_ptr(), db.data_ptr(), dz.data_ptr(), ws.data_ptr(),
                           ws.numel(), N.BF16, s)
torch.cuda.synchronize()
print("ok")
