"""Per-launch GPU time (CUDA graph, 20 launches) of the LayerNorm and
BatchNorm C-ABI ops at the bench geometries, with algorithmic GB/s.
usage: python tools/norm_graph.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_2411_12780_b200 import _native as N
from gemm_graph import per_launch  # noqa: E402

lib = N.load()
bf = torch.bfloat16


def ln(M, D):
    x, dy, dres = (torch.randn(M, D, device="cuda").to(bf) for _ in range(3))
    y, dx = torch.empty_like(x), torch.empty_like(x)
    g, b = torch.ones(D, device="cuda"), torch.zeros(D, device="cuda")
    mean, rstd = torch.empty(M, device="cuda"), torch.empty(M, device="cuda")
    dg, db, dxs = (torch.empty(D, device="cuda") for _ in range(3))
    ws = torch.empty(lib.ppll_layernorm_bwd_ws_floats(M, D), device="cuda")
    f = lambda s: lib.ppll_layernorm_fwd(M, D, x.data_ptr(), D, g.data_ptr(), b.data_ptr(),  # noqa
                                         y.data_ptr(), D, mean.data_ptr(), rstd.data_ptr(), N.BF16, s)
    f(torch.cuda.current_stream().cuda_stream)
    bw = lambda s: lib.ppll_layernorm_bwd(M, D, dy.data_ptr(), D, x.data_ptr(), D,  # noqa
                                          mean.data_ptr(), rstd.data_ptr(), g.data_ptr(),
                                          dres.data_ptr(), D, dx.data_ptr(), D, dg.data_ptr(),
                                          db.data_ptr(), dxs.data_ptr(), ws.data_ptr(), ws.numel(),
                                          N.BF16, s)
    for name, fn, by in (("ln fwd", f, 4 * M * D), ("ln bwd (+res, +dxsum)", bw, 8 * M * D)):
        us = per_launch(fn)
        print(f"{name:24s} M={M} D={D}: {us:6.2f} us  {by / us / 1e3:6.0f} GB/s algorithmic")


def bnorm(P, C):
    z, dy = torch.randn(P, C, device="cuda").to(bf), torch.randn(P, C, device="cuda").to(bf)
    y, dz = torch.empty_like(z), torch.empty_like(z)
    g, b = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
    mean, rstd, dg, db = (torch.empty(C, device="cuda") for _ in range(4))
    ws = torch.empty(lib.ppll_batchnorm_ws_floats(P, C), device="cuda")
    f = lambda s: lib.ppll_batchnorm_fwd(P, C, z.data_ptr(), g.data_ptr(), b.data_ptr(), None, 1,  # noqa
                                         y.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                         ws.data_ptr(), ws.numel(), N.BF16, s)
    bw = lambda s: lib.ppll_batchnorm_bwd(P, C, dy.data_ptr(), z.data_ptr(), mean.data_ptr(),  # noqa
                                          rstd.data_ptr(), g.data_ptr(), dg.data_ptr(), db.data_ptr(),
                                          dz.data_ptr(), ws.data_ptr(), ws.numel(), N.BF16, s)
    for name, fn, by in (("bn fwd (stats+apply)", f, 6 * P * C), ("bn bwd", bw, 8 * P * C)):
        us = per_launch(fn)
        print(f"{name:24s} P={P} C={C}: {us:6.2f} us  {by / us / 1e3:6.0f} GB/s algorithmic")


ln(8320, 384)
for P, C in ((131072, 16), (32768, 32), (8192, 64), (262144, 16), (524288, 16)):
    bnorm(P, C)
