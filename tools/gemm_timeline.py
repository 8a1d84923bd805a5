"""Per-tile timeline of one tcgen05 GEMM launch (PPLL_GEMM_TIMELINE=1):
MMA duration per tile, epilogue duration per tile, and how long the MMA
waited for a free accumulator (epilogue-bound) — averaged over CTAs.

usage: PPLL_GEMM_TIMELINE=1 python tools/gemm_timeline.py M K N [fwd|fwdgelu|dgrad|dgradmul]
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2411_12780_b200 import _native as N

M, K, Nn = (int(v) for v in sys.argv[1:4])
op = sys.argv[4] if len(sys.argv) > 4 else "fwd"
lib = N.load()
s = torch.cuda.current_stream().cuda_stream
X = torch.randn(M, K, device="cuda").bfloat16()
W = (torch.randn(K, Nn, device="cuda") * 0.05).bfloat16()
b = torch.zeros(Nn, device="cuda")
Y = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
P = torch.empty_like(Y)
dY = torch.randn(M, Nn, device="cuda").bfloat16()
dX = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
Mk = torch.rand(M, K, device="cuda").bfloat16()
fns = {
    "fwd": lambda: lib.ppll_linear_fwd_ex(M, K, Nn, X.data_ptr(), K, W.data_ptr(), b.data_ptr(),
                                          None, 0, 0, None, 0, Y.data_ptr(), Nn, None, 0, N.BF16, s),
    "fwdgelu": lambda: lib.ppll_linear_fwd_ex(M, K, Nn, X.data_ptr(), K, W.data_ptr(),
                                              b.data_ptr(), None, 0, 3, P.data_ptr(), Nn,
                                              Y.data_ptr(), Nn, None, 0, N.BF16, s),
    "dgrad": lambda: lib.ppll_linear_dgrad_ex(M, K, Nn, dY.data_ptr(), Nn, W.data_ptr(), None, 0,
                                              0, dX.data_ptr(), K, N.BF16, s),
    "dgradmul": lambda: lib.ppll_linear_dgrad_ex(M, K, Nn, dY.data_ptr(), Nn, W.data_ptr(),
                                                 Mk.data_ptr(), K, 3, dX.data_ptr(), K, N.BF16, s),
}
fn = fns[op]
for _ in range(3):
    fn()
torch.cuda.synchronize()
buf = lib.ppll_gemm_timeline()
host = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
zero = torch.zeros_like(host)
N.check(lib.ppll_copy_async(buf, zero.data_ptr(), host.numel() * 8, s), "zero")
fn()
N.check(lib.ppll_copy_async(host.data_ptr(), buf, host.numel() * 8, s), "copy")
torch.cuda.synchronize()
t = host.cpu().numpy().reshape(148, 4, 4).astype(np.float64)
valid = t[:, :, 0] > 0
t0 = t[:, :, 0][valid].min()
mma = (t[:, :, 1] - t[:, :, 0])[valid]
epi = (t[:, :, 2] - t[:, :, 1])[valid]
# gap between a tile's MMA start and the previous tile's MMA done (waiting for a free accumulator)
ends = t[:, :, 2][valid]
print(f"{op} M={M} K={K} N={Nn}: tiles/CTA max {valid.sum(1).max()}, "
      f"kernel span {(ends.max() - t0) / 1e3:.2f} us from first MMA start")
print(f"  MMA phase per tile  mean {mma.mean() / 1e3:.2f} us  max {mma.max() / 1e3:.2f}")
print(f"  epilogue per tile   mean {epi.mean() / 1e3:.2f} us  max {epi.max() / 1e3:.2f}")
first = t[:, 0, 0][t[:, 0, 0] > 0]
print(f"  first MMA start spread {(first.max() - first.min()) / 1e3:.2f} us; "
      f"first-tile MMA {np.mean(t[:, 0, 1][t[:, 0, 0] > 0] - first) / 1e3:.2f} us")
