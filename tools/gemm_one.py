"""Run one linear-layer GEMM shape through the C-ABI (for ncu captures / probes).

usage: python tools/gemm_one.py M K N [fwd|fwdgelu|dgrad|dgradmul|wgrad] [iters]
  fwdgelu : bias + GELU, gelu'(pre-activation) stored (the ViT FC1 forward)
  dgradmul: dX = (dY·Wᵀ) ∘ mask (the ViT FC2 dgrad with the stored derivative)
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_12780_b200 import _native as N

M, K, Nn = (int(v) for v in sys.argv[1:4])
op = sys.argv[4] if len(sys.argv) > 4 else "fwd"
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 5
lib = N.load()
s = torch.cuda.current_stream().cuda_stream
X = torch.randn(M, K, device="cuda").bfloat16()
W = (torch.randn(K, Nn, device="cuda") * 0.05).bfloat16()
b = torch.zeros(Nn, device="cuda")
Y = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
dY = torch.randn(M, Nn, device="cuda").bfloat16()
dX = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
dW = torch.empty(K, Nn, device="cuda")
if op == "fwd":
    fn = lambda: lib.ppll_linear_fwd(M, K, Nn, X.data_ptr(), K, W.data_ptr(), b.data_ptr(),
                                     Y.data_ptr(), Nn, None, 0, 1, N.BF16, s)
elif op == "fwdgelu":
    P = torch.empty_like(Y)
    fn = lambda: lib.ppll_linear_fwd_ex(M, K, Nn, X.data_ptr(), K, W.data_ptr(), b.data_ptr(),
                                        None, 0, 3, P.data_ptr(), Nn, Y.data_ptr(), Nn, None, 0,
                                        N.BF16, s)
elif op == "dgradmul":
    Mk = torch.rand(M, K, device="cuda").bfloat16()
    fn = lambda: lib.ppll_linear_dgrad_ex(M, K, Nn, dY.data_ptr(), Nn, W.data_ptr(),
                                          Mk.data_ptr(), K, 3, dX.data_ptr(), K, N.BF16, s)
elif op == "dgrad":
    fn = lambda: lib.ppll_linear_dgrad(M, K, Nn, dY.data_ptr(), Nn, W.data_ptr(), None, 0,
                                       dX.data_ptr(), K, N.BF16, s)
else:
    fn = lambda: lib.ppll_linear_wgrad(M, K, Nn, X.data_ptr(), K, dY.data_ptr(), Nn,
                                       dW.data_ptr(), None, N.BF16, s)
for _ in range(3):
    fn()
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(iters):
    fn()
e.record()
torch.cuda.synchronize()
t = a.elapsed_time(e) / iters
print(f"{op} M={M} K={K} N={Nn}: {t * 1e3:.1f} us  {2.0 * M * K * Nn / t / 1e9:.0f} TF/s")
# correctness against torch (fp32 accumulate of the same bf16 operands)
if op in ("fwd", "dgrad"):
    fn()
    torch.cuda.synchronize()
    if op == "fwd":
        ref, got = (X.float() @ W.float() + b).clamp_min(0), Y.float()   # bias + ReLU
    else:
        ref, got = dY.float() @ W.float().t(), dX.float()
    err = ((got - ref).abs().max() / ref.abs().max()).item()
    print(f"  max rel err vs torch: {err:.2e}")
