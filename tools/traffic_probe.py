"""One launch of every kernel a bench.py roofline entry names, at the bench
geometry, for the ncu DRAM-traffic capture bench.py attaches as `traffic`
(profiles/r02_ncu_traffic.csv):

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file profiles/r02_ncu_traffic.csv \
      python tools/traffic_probe.py

Kernels, in launch order: attention forward + backward (ViT-S, B=128 T=65
H=6), the implicit conv forward at the three ResNet-32 resolutions (batch
128), the fused Nesterov update (ResNet-32's largest stage, 373,056 params,
bf16 shadow).  ncu flushes the caches before every launch, so each row is the
cold-cache DRAM traffic of one launch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_12780_b200 import _native as N

lib = N.load()
s = torch.cuda.current_stream().cuda_stream

B, T, H = 128, 65, 6
D = 64 * H
qkv = torch.randn(B * T, 3 * D, device="cuda").bfloat16()
dout = torch.randn(B * T, D, device="cuda").bfloat16()
o = torch.empty(B * T, D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * T, device="cuda")
dqkv = torch.empty(B * T, 3 * D, device="cuda", dtype=torch.bfloat16)
bp = torch.empty(B, 3 * D, device="cuda")
N.check(lib.ppll_attn_fwd_bf16(B, T, H, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), s), "attn fwd")
N.check(lib.ppll_attn_bwd_bf16(B, T, H, qkv.data_ptr(), o.data_ptr(), dout.data_ptr(),
                               lse.data_ptr(), dqkv.data_ptr(), bp.data_ptr(), s), "attn bwd")

for C, HW in ((16, 32), (32, 16), (64, 8)):
    x = torch.randn(128, HW, HW, C, device="cuda").bfloat16()
    w = (torch.randn(9 * C, C, device="cuda") * 0.05).bfloat16()
    y = torch.empty_like(x)
    N.check(lib.ppll_conv3x3_bf16(128, HW, HW, C, C, x.data_ptr(), w.data_ptr(), y.data_ptr(), 0, s),
            "conv")

n = 373056
th = torch.randn(n, device="cuda")
v = torch.zeros(n, device="cuda")
g = torch.randn(n, device="cuda")
lp = torch.empty(n, device="cuda", dtype=torch.bfloat16)
N.check(lib.ppll_nesterov_step(n, th.data_ptr(), v.data_ptr(), g.data_ptr(), lp.data_ptr(), None,
                               None, 0, 0.01, 0.9, 1e-4, None, s), "nesterov")
torch.cuda.synchronize()
print("traffic probe done")
