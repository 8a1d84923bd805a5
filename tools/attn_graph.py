"""Per-launch GPU time of the attention kernels in a CUDA graph (20 launches,
replayed), ViT-S geometry by default.  usage: python tools/attn_graph.py [B T H]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_12780_b200 import _native as N
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_graph import per_launch  # noqa: E402

B, T, H = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (128, 65, 6)
D = 64 * H
lib = N.load()
qkv = torch.randn(B * T, 3 * D, device="cuda").bfloat16()
dout = torch.randn(B * T, D, device="cuda").bfloat16()
o = torch.empty(B * T, D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * T, device="cuda")
dqkv = torch.empty(B * T, 3 * D, device="cuda", dtype=torch.bfloat16)
bp = torch.empty(B, 3 * D, device="cuda")
fwd = lambda s: lib.ppll_attn_fwd_bf16(B, T, H, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), s)  # noqa
bwd = lambda s: lib.ppll_attn_bwd_bf16(B, T, H, qkv.data_ptr(), o.data_ptr(), dout.data_ptr(),  # noqa
                                       lse.data_ptr(), dqkv.data_ptr(), bp.data_ptr(), s)
byf = 2 * B * T * (3 * D + D)                 # qkv in, o out (+ lse)
byb = 2 * B * T * (3 * D + 2 * D + 3 * D)     # qkv, o, dout in; dqkv out
for name, fn, by in (("fwd", fwd, byf), ("bwd", bwd, byb)):
    us = per_launch(fn)
    print(f"attn {name} B={B} T={T} H={H}: {us:6.2f} us/launch in a graph, "
          f"{by / us / 1e3:6.0f} GB/s algorithmic")
