"""One shape of the implicit conv weight gradient, a few launches, for ncu.
usage: python tools/wgrad_one.py C H exclusive(0|1) [batch]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_12780_b200 import _native as N

C, H, excl = (int(v) for v in sys.argv[1:4])
B = int(sys.argv[4]) if len(sys.argv) > 4 else 128
lib = N.load()
x = torch.randn(B, H, H, C, device="cuda").bfloat16()
dz = torch.randn(B, H, H, C, device="cuda").bfloat16()
nws = lib.ppll_conv3x3_wgrad_ws_floats(B, H, H, C, C)
ws = torch.empty(nws, device="cuda")
dw = torch.empty(9 * C, C, device="cuda")
lib.ppll_set_gpu_exclusive(excl)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    N.check(lib.ppll_conv3x3_wgrad_bf16(B, H, H, C, C, x.data_ptr(), dz.data_ptr(), dw.data_ptr(),
                                        ws.data_ptr(), nws, s), "wgrad")
torch.cuda.synchronize()
print("ok")
