"""Phase timeline of the fused GEMM + LayerNorm-backward kernel inside one ViT
stage step (PPLL_GEMM_LN_TIMELINE=1): per CTA %globaltimer at start / all MMAs
retired / x, dres tiles landed / row sums done / column sums done (µs).
usage: PPLL_GEMM_LN_TIMELINE=1 PPLL_PDL=0 python tools/gln_timeline.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import torch
import cuda.bindings.runtime as rt
import paper_2411_12780_b200 as lp
from paper_2411_12780_b200 import _native as N

lib = N.load()
lib.ppll_gemm_timeline.restype = ctypes.c_void_p
buf = lib.ppll_gemm_timeline()
torch.cuda.set_device(0)
hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=10 ** 6, seed=1, precision="bf16")
spec = lp.VitSpec()
mods = lp.build_vit_modules(spec, lp.balanced_depths(spec.depth, 4), 1, 3, hyper)
m = mods[3]
B = 128
x = torch.randn((B,) + tuple(m.in_shape), device="cuda").to(m.act_dtype)
y = torch.as_tensor(np.random.default_rng(0).integers(0, 10, B), device="cuda")
out = torch.empty((B,) + tuple(m.out_shape), device="cuda", dtype=m.act_dtype)
m.native(B)
s = torch.cuda.current_stream()
for _ in range(3):
    m.launch_step(B, x.data_ptr(), y.data_ptr(), out.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
rt.cudaMemset(buf, 0, 65536 * 8)
m.launch_step(B, x.data_ptr(), y.data_ptr(), out.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
host = np.zeros(130 * 8, dtype=np.uint64)
rt.cudaMemcpy(host.ctypes.data, buf, host.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
a = host.reshape(130, 8)[:, :5].astype(np.float64)
a = a[a[:, 0] > 0]
rel = (a - a[:, 0].min()) / 1e3
names = ["start", "mma done", "x/dres", "row sums", "col sums"]
print(f"{len(a)} CTAs (last launch of the step): " + "  ".join(
    f"{n} {rel[:, k].mean():.2f} [{rel[:, k].min():.2f},{rel[:, k].max():.2f}]" for k, n in enumerate(names)))
