"""Drive a few ViT-S stage steps (bf16) + standalone FC1 GEMMs for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2411_12780_b200 as lp
from paper_2411_12780_b200 import _native as N

torch.cuda.set_device(0)
spec = lp.VitSpec()
hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=100, seed=1, precision="bf16")
mods = lp.build_vit_modules(spec, [2, 2, 2, 2], 1, 3, hyper)
x = lp.Tensor(torch.randn(128, 3, 32, 32, device="cuda"))
y = np.random.default_rng(0).integers(0, 10, 128)
for _ in range(3):
    h = x
    for m in mods[:2]:
        _, h = lp.local_loss_and_update(m, h, y)
M, K, Nn = 8320, 384, 1536
X = torch.randn(M, K, device="cuda").bfloat16()
W = (torch.randn(K, Nn, device="cuda") * 0.05).bfloat16()
b = torch.zeros(Nn, device="cuda")
Y = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
lib = N.load()
for _ in range(3):
    lib.ppll_linear_fwd(M, K, Nn, X.data_ptr(), K, W.data_ptr(), b.data_ptr(), Y.data_ptr(), Nn,
                        None, 0, 1, N.BF16, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("done")
