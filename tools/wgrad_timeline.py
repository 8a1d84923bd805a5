"""Phase timeline of one cluster split-K weight-gradient launch
(gemm_tc_cluster_kernel, PPLL_GEMM_TIMELINE=1): per CTA %globaltimer at
start (after griddepcontrol.wait), first operands landed, mainloop done,
partial dumped + cluster barrier, reduction done, exit — mean / max over CTAs
relative to the earliest CTA start.

usage: PPLL_GEMM_TIMELINE=1 python tools/wgrad_timeline.py M K N
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2411_12780_b200 import _native as N

M, K, Nn = (int(v) for v in sys.argv[1:4])
lib = N.load()
s = torch.cuda.current_stream().cuda_stream
X = torch.randn(M, K, device="cuda").bfloat16()
dY = torch.randn(M, Nn, device="cuda").bfloat16()
dW = torch.empty(K, Nn, device="cuda")
fn = lambda: lib.ppll_linear_wgrad(M, K, Nn, X.data_ptr(), K, dY.data_ptr(), Nn, dW.data_ptr(),  # noqa
                                   None, N.BF16, s)
for _ in range(3):
    fn()
torch.cuda.synchronize()
buf = lib.ppll_gemm_timeline()
host = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
zero = torch.zeros_like(host)
names = ["start", "operands", "mainloop", "dump+barrier", "reduced", "exit"]
acc = []
for rep in range(5):
    N.check(lib.ppll_copy_async(buf, zero.data_ptr(), host.numel() * 8, s), "zero")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    N.check(lib.ppll_copy_async(host.data_ptr(), buf, host.numel() * 8, s), "copy")
    torch.cuda.synchronize()
    t = host.cpu().numpy().reshape(148 * 2, 8)[:, :6].astype(np.float64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    acc.append(((t - t0) / 1e3, a.elapsed_time(b) * 1e3))
ref = X.float().t() @ dY.float()
err = ((dW - ref).abs().max() / ref.abs().max()).item()
ctas = acc[-1][0].shape[0]
print(f"  max rel err vs torch: {err:.2e}")
print(f"wgrad M={M} K={K} N={Nn}: {ctas} CTAs, event time {np.mean([e for _, e in acc]):.2f} us")
for i, n in enumerate(names):
    m = np.mean([x[:, i].mean() for x, _ in acc])
    mx = np.mean([x[:, i].max() for x, _ in acc])
    print(f"  {n:13s} mean {m:6.2f} us   max {mx:6.2f} us")
