"""Phase timeline of the fused single-cluster BatchNorm kernels
(PPLL_BN_TIMELINE=1): per CTA %globaltimer at entry / after the grid
dependency wait / statistics pass / CTA merge / cluster merge / apply pass /
exit, relative to the earliest entry, in µs.
usage: PPLL_BN_TIMELINE=1 python tools/bn_timeline.py P C"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import torch
from paper_2411_12780_b200 import _native as N

lib = N.load()
P, C = int(sys.argv[1]), int(sys.argv[2])
bf = torch.bfloat16
z, dy = torch.randn(P, C, device="cuda").to(bf), torch.randn(P, C, device="cuda").to(bf)
y, dz = torch.empty_like(z), torch.empty_like(z)
g, b = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
mean, rstd, dg, db = (torch.empty(C, device="cuda") for _ in range(4))
ws = torch.empty(lib.ppll_batchnorm_ws_floats(P, C), device="cuda")
s = torch.cuda.current_stream().cuda_stream
lib.ppll_gemm_timeline.restype = ctypes.c_void_p
buf = lib.ppll_gemm_timeline()
names = ["entry", "pdl", "stats", "cta-merge", "cl-merge", "apply", "exit", "cl-sync"]
for which in ("fwd", "bwd"):
    for it in range(3):
        if which == "fwd":
            lib.ppll_batchnorm_fwd(P, C, z.data_ptr(), g.data_ptr(), b.data_ptr(), None, 1,
                                   y.data_ptr(), mean.data_ptr(), rstd.data_ptr(), ws.data_ptr(),
                                   ws.numel(), N.BF16, s)
        else:
            lib.ppll_batchnorm_bwd(P, C, dy.data_ptr(), z.data_ptr(), mean.data_ptr(),
                                   rstd.data_ptr(), g.data_ptr(), dg.data_ptr(), db.data_ptr(),
                                   dz.data_ptr(), ws.data_ptr(), ws.numel(), N.BF16, s)
        torch.cuda.synchronize()
    t = torch.empty(16 * 8, dtype=torch.int64, device="cuda")
    ctypes.memmove(ctypes.c_void_p(0), 0, 0) if False else None
    torch.cuda.synchronize()
    host = np.zeros(16 * 8, dtype=np.uint64)
    import cuda.bindings.runtime as rt  # noqa
    rt.cudaMemcpy(host.ctypes.data, buf, host.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    a = host.reshape(16, 8)[:, :8].astype(np.float64)
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    rel = (a - t0) / 1e3
    print(f"{which} P={P} C={C} ({len(a)} CTAs): " +
          "  ".join(f"{n} {rel[:, k].mean():.2f} [{rel[:, k].min():.2f},{rel[:, k].max():.2f}]"
                    for k, n in enumerate(names)))
