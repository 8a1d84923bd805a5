"""Per-item phase timeline of the persistent attention backward
(PPLL_ATTN_TIMELINE=1): mean over CTAs of the first items' stamps (µs) —
start, inputs landed, S/dP retired, P/dS stored, dV/dK/dQ retired, done.
usage: PPLL_ATTN_TIMELINE=1 python tools/attn_timeline.py [B T H]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import torch
from paper_2411_12780_b200 import _native as N
import cuda.bindings.runtime as rt

B, T, H = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (128, 65, 6)
D = 64 * H
lib = N.load()
lib.ppll_gemm_timeline.restype = ctypes.c_void_p
buf = lib.ppll_gemm_timeline()
qkv = torch.randn(B * T, 3 * D, device="cuda").bfloat16()
dout = torch.randn(B * T, D, device="cuda").bfloat16()
o = torch.empty(B * T, D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * T, device="cuda")
dqkv = torch.empty_like(qkv)
s = torch.cuda.current_stream().cuda_stream
lib.ppll_attn_fwd_bf16(B, T, H, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), s)
for _ in range(3):
    torch.cuda.synchronize()
    rt.cudaMemset(buf, 0, 65536 * 8)
    lib.ppll_attn_bwd_bf16(B, T, H, qkv.data_ptr(), o.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                           dqkv.data_ptr(), None, s)
    torch.cuda.synchronize()
host = np.zeros(65536, dtype=np.uint64)
rt.cudaMemcpy(host.ctypes.data, buf, host.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
a = host[: 2048 * 32].reshape(-1, 4, 8)[:, :, :6].astype(np.float64)
ctas = a[a[:, 0, 0] > 0]
t0 = ctas[:, 0, 0].min()
names = ["start", "loaded", "S/dP", "P/dS", "dQKV mma", "done"]
print(f"B={B} T={T} H={H}: {len(ctas)} CTAs, end {(ctas[ctas > 0].max() - t0) / 1e3:.2f} us")
for it in range(4):
    x = ctas[:, it, :]
    x = x[x[:, 0] > 0]
    if not len(x):
        break
    rel = (x - t0) / 1e3
    d = np.diff(rel, axis=1).mean(axis=0)
    print(f" item {it} ({len(x)} CTAs): start {rel[:, 0].mean():.2f} [{rel[:, 0].min():.2f},{rel[:, 0].max():.2f}]  "
          + "  ".join(f"{names[k + 1]} +{d[k]:.2f}" for k in range(5)) + f"  end {rel[:, 5].mean():.2f}")
