"""LayerNorm and train-mode BatchNorm kernels through the C-ABI
(ppll_layernorm_fwd/bwd, ppll_batchnorm_fwd/bwd) against float64 torch
autograd on the same inputs, at the ViT-S (8320 tokens x 384) and ResNet-32
(NHWC 128x32x32x16, 128x8x8x64) geometries plus ragged sizes.

Tolerances: fp32 — outputs / input gradients 2e-4 of max, parameter gradients
2e-4 relative; bf16 (activations stored bf16, statistics fp32) — 1.5e-2 of
max, parameter gradients 1e-2 relative."""
import pytest
import torch
import torch.nn.functional as F

from paper_2411_12780_b200 import _native as N

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _rel(a, b):
    return ((a.double() - b.double()).abs().max() / b.double().abs().max()).item()


TOL = {"fp32": (2e-4, 2e-4), "bf16": (1.5e-2, 1e-2)}


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("M,D", [(8320, 384), (37, 128), (1000, 768), (130, 96)])
def test_layernorm_matches_torch(precision, M, D):
    dt = torch.float32 if precision == "fp32" else torch.bfloat16
    code = N.F32 if precision == "fp32" else N.BF16
    g = torch.Generator(device="cuda").manual_seed(M + D)
    x = (torch.randn(M, D, device="cuda", generator=g) * 2 + 0.5).to(dt)
    dy = torch.randn(M, D, device="cuda", generator=g).to(dt)
    dres = torch.randn(M, D, device="cuda", generator=g).to(dt)
    gam = torch.rand(D, device="cuda", generator=g) + 0.5
    bet = torch.randn(D, device="cuda", generator=g) * 0.1
    y = torch.empty(M, D, device="cuda", dtype=dt)
    dx = torch.empty(M, D, device="cuda", dtype=dt)
    mean, rstd = torch.empty(M, device="cuda"), torch.empty(M, device="cuda")
    dg, db, dxs = (torch.empty(D, device="cuda") for _ in range(3))
    lib = N.load()
    ws = torch.empty(lib.ppll_layernorm_bwd_ws_floats(M, D), device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    N.check(lib.ppll_layernorm_fwd(M, D, x.data_ptr(), D, gam.data_ptr(), bet.data_ptr(),
                                   y.data_ptr(), D, mean.data_ptr(), rstd.data_ptr(), code, s), "fwd")
    N.check(lib.ppll_layernorm_bwd(M, D, dy.data_ptr(), D, x.data_ptr(), D, mean.data_ptr(),
                                   rstd.data_ptr(), gam.data_ptr(), dres.data_ptr(), D,
                                   dx.data_ptr(), D, dg.data_ptr(), db.data_ptr(), dxs.data_ptr(),
                                   ws.data_ptr(), ws.numel(), code, s), "bwd")
    torch.cuda.synchronize()
    xr = x.double().requires_grad_(True)
    gr, br = gam.double().requires_grad_(True), bet.double().requires_grad_(True)
    yr = F.layer_norm(xr, (D,), gr, br, 1e-5)
    yr.backward(dy.double())
    ta, tp = TOL[precision]
    assert _rel(y, yr) < ta
    assert _rel(mean, xr.detach().mean(1)) < 1e-5
    ref_dx = xr.grad + dres.double()
    assert _rel(dx, ref_dx) < ta
    assert _rel(dg, gr.grad) < tp and _rel(db, br.grad) < tp
    # the fused Σ rows of the dx output (bias gradient of the layer below)
    assert _rel(dxs, dx.double().sum(0) if precision == "fp32" else ref_dx.sum(0)) < tp


@pytest.mark.parametrize("exclusive", [1, 0])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("P,C,res", [(131072, 16, False), (8192, 64, True), (2048, 32, True),
                                     (300, 24, False), (131072, 16, True), (262144, 32, False),
                                     (524288, 16, True), (1048576, 16, False)])
def test_batchnorm_matches_torch(precision, P, C, res, exclusive):
    """exclusive = 1: large bf16 tensors take the cooperative full-GPU form;
    0 (stage streams sharing the GPU): the two-launch split form."""
    prev = N.load().ppll_set_gpu_exclusive(exclusive)
    try:
        _batchnorm_case(precision, P, C, res)
    finally:
        N.load().ppll_set_gpu_exclusive(prev)


def _batchnorm_case(precision, P, C, res):
    dt = torch.float32 if precision == "fp32" else torch.bfloat16
    code = N.F32 if precision == "fp32" else N.BF16
    g = torch.Generator(device="cuda").manual_seed(P + C)
    z = (torch.randn(P, C, device="cuda", generator=g) * 3 - 1).to(dt)
    r = torch.randn(P, C, device="cuda", generator=g).to(dt) if res else None
    dy = torch.randn(P, C, device="cuda", generator=g).to(dt)
    gam = torch.rand(C, device="cuda", generator=g) + 0.5
    bet = torch.randn(C, device="cuda", generator=g) * 0.1
    y, dz = torch.empty(P, C, device="cuda", dtype=dt), torch.empty(P, C, device="cuda", dtype=dt)
    mean, rstd, dg, db = (torch.empty(C, device="cuda") for _ in range(4))
    lib = N.load()
    ws = torch.empty(lib.ppll_batchnorm_ws_floats(P, C), device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    N.check(lib.ppll_batchnorm_fwd(P, C, z.data_ptr(), gam.data_ptr(), bet.data_ptr(),
                                   N.ptr(r), 1, y.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                   ws.data_ptr(), ws.numel(), code, s), "bn fwd")
    N.check(lib.ppll_batchnorm_bwd(P, C, dy.data_ptr(), z.data_ptr(), mean.data_ptr(),
                                   rstd.data_ptr(), gam.data_ptr(), dg.data_ptr(), db.data_ptr(),
                                   dz.data_ptr(), ws.data_ptr(), ws.numel(), code, s), "bn bwd")
    torch.cuda.synchronize()
    zr = z.double().requires_grad_(True)
    gr, br = gam.double().requires_grad_(True), bet.double().requires_grad_(True)
    bn = F.batch_norm(zr, None, None, gr, br, training=True, eps=1e-5)
    out = torch.relu(bn + (r.double() if res else 0.0))
    ta, tp = TOL[precision]
    assert _rel(y, out) < ta
    assert _rel(mean, zr.detach().mean(0)) < 1e-5
    bn.backward(dy.double())            # the kernel's backward starts after the ReLU / residual
    assert _rel(dz, zr.grad) < ta
    assert _rel(dg, gr.grad) < tp and _rel(db, br.grad) < tp


def test_norm_workspace_is_checked():
    lib = N.load()
    assert lib.ppll_layernorm_bwd(64, 128, 1, 128, 1, 128, 1, 1, 1, None, 0, None, 0, None, None,
                                  None, 1, 10, N.BF16, None) != 0
    assert lib.ppll_batchnorm_bwd(64, 16, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, N.BF16, None) != 0
