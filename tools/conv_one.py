"""One implicit-GEMM 3x3 convolution launch (for ncu): python tools/conv_one.py N H C [dgrad]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2411_12780_b200 import _native as N

n, h, c = (int(v) for v in sys.argv[1:4])
dg = int(sys.argv[4]) if len(sys.argv) > 4 else 0
lib = N.load()
x = torch.randn(n, h, h, c, device="cuda").bfloat16()
w = (torch.randn(9 * c, c, device="cuda") * 0.05).bfloat16()
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    N.check(lib.ppll_conv3x3_bf16(n, h, h, c, c, x.data_ptr(), w.data_ptr(), y.data_ptr(), dg, s))
torch.cuda.synchronize()
print("ok")
