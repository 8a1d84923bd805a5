"""Micro-benchmark of the linear-layer engines vs torch (cuBLAS) on one GPU."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_12780_b200 import _native as N

def bench(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / iters

lib = N.load()
s = torch.cuda.current_stream().cuda_stream
shapes = [(8192, 8192, 8192), (8320, 384, 1152), (8320, 384, 1536), (8320, 1536, 384),
          (128, 3072, 1024), (128, 1024, 1024), (4736, 768, 3072)]
for M, K, Nn in shapes:
    X = torch.randn(M, K, device="cuda").bfloat16()
    W = torch.randn(K, Nn, device="cuda").bfloat16() * 0.02
    b = torch.zeros(Nn, device="cuda")
    Y = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
    dY = torch.randn(M, Nn, device="cuda").bfloat16()
    dX = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
    dW = torch.empty(K, Nn, device="cuda")
    fl = 2.0 * M * K * Nn
    t_f = bench(lambda: lib.ppll_linear_fwd(M, K, Nn, X.data_ptr(), K, W.data_ptr(), b.data_ptr(), Y.data_ptr(), Nn, None, 0, 1, N.BF16, s))
    t_d = bench(lambda: lib.ppll_linear_dgrad(M, K, Nn, dY.data_ptr(), Nn, W.data_ptr(), None, 0, dX.data_ptr(), K, N.BF16, s))
    t_w = bench(lambda: lib.ppll_linear_wgrad(M, K, Nn, X.data_ptr(), K, dY.data_ptr(), Nn, dW.data_ptr(), None, N.BF16, s))
    t_t = bench(lambda: torch.matmul(X, W))
    t_tw = bench(lambda: torch.matmul(X.T, dY))
    print(f"M={M} K={K} N={Nn}: fwd {fl/t_f/1e9:.0f} TF/s ({t_f*1e3:.1f}us)  dgrad {fl/t_d/1e9:.0f}  wgrad {fl/t_w/1e9:.0f}  | torch fwd {fl/t_t/1e9:.0f} wgrad {fl/t_tw/1e9:.0f}", flush=True)
