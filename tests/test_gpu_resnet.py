"""GPU parity of the ResNet local step (native ``ppll_resnet_stage_step``)
against the float64 CPU restatement ``oracle/resnet_oracle.py`` (pinned to
torch autograd in tests/test_resnet_oracle.py).

Tolerances: fp32 parity mode — per-step loss |Δ| <= 2e-4·max(1,|loss|),
x_out max|Δ|/max|ref| <= 2e-4, weights max|ΔW|/max|W| <= 2e-3; bf16 mode
— loss 5e-2 relative, x_out 8e-2, weights 8e-2 (BatchNorm over bf16
activations).  Pipeline vs round-robin: bitwise."""
import os

import numpy as np
import pytest
import torch

import paper_2411_12780_b200 as lp
import resnet_oracle as ro

pytestmark = pytest.mark.gpu

SMALL = dict(n=1, image=8, channels=3, widths=(16, 32, 64), classes=5)


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _pair(kw, s, d_prime, n, precision, steps, seed=7):
    hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=steps, seed=seed, precision=precision)
    mods = lp.build_resnet_modules(lp.ResNetSpec(**kw), s, d_prime, n, hyper)
    stages = ro.build_resnet_stages(ro.ResNetSpec(**kw), s, d_prime, n, seed)
    return mods, stages


def _flat(m):
    return np.concatenate([p.data.ravel() for p in m.parameters()])


def _flat_o(st):
    return np.concatenate([p.ravel() for p in st.params()])


def test_init_matches_oracle():
    mods, stages = _pair(SMALL, 3, 1, 2, "fp32", 4)
    assert [m.n_aux_convs for m in mods] == [len(s.aux) for s in stages]
    for m, st in zip(mods, stages):
        np.testing.assert_allclose(_flat(m), _flat_o(st), rtol=0, atol=1e-7)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_resnet_local_steps_match_oracle(precision):
    steps = 3
    mods, stages = _pair(SMALL, 3, 1, 2, precision, steps)
    rng = np.random.default_rng(0)
    B = 8
    ltol, xtol, wtol = (2e-4, 2e-4, 2e-3) if precision == "fp32" else (5e-2, 8e-2, 8e-2)
    for t in range(steps):
        img = rng.standard_normal((B, 8, 8, 3))
        y = rng.integers(0, 5, B)
        h, hr = lp.Tensor(img), img
        for j, (m, st) in enumerate(zip(mods, stages)):
            loss, h = lp.local_loss_and_update(m, h, y)
            ref, hr, _ = ro.local_step(st, hr, y, 0.05, 0.001, steps, 0.9, 1e-4)
            assert abs(loss - ref) <= ltol * max(1.0, abs(ref)), (t, j, loss, ref)
            hd = h.data.reshape(hr.shape)
            assert np.abs(hd - hr).max() / np.abs(hr).max() <= xtol, (t, j)
            hr = hd if precision == "bf16" else hr
    for m, st in zip(mods, stages):
        a, b = _flat(m), _flat_o(st)
        assert np.abs(a - b).max() / np.abs(b).max() <= wtol


def test_resnet32_geometry_one_step_fp32():
    """ResNet-32 split into 4 stages, batch 4, one step of every stage."""
    kw = dict(n=5, image=32, channels=3, widths=(16, 32, 64), classes=10)
    mods, stages = _pair(kw, 4, 2, 3, "fp32", 2)
    assert [len(m.block_ids) for m in mods] == [3, 4, 4, 4]
    rng = np.random.default_rng(1)
    img = rng.standard_normal((4, 32, 32, 3))
    y = np.array([3, 7, 1, 0])
    h, hr = lp.Tensor(img), img
    for m, st in zip(mods, stages):
        loss, h = lp.local_loss_and_update(m, h, y)
        ref, hr, _ = ro.local_step(st, hr, y, 0.05, 0.001, 2, 0.9, 1e-4)
        assert abs(loss - ref) <= 2e-4 * max(1.0, abs(ref))
        assert np.abs(h.data.reshape(hr.shape) - hr).max() / np.abs(hr).max() <= 2e-4
    for m, st in zip(mods, stages):
        a, b = _flat(m), _flat_o(st)
        assert np.abs(a - b).max() / np.abs(b).max() <= 2e-3


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_resnet_pipeline_bitwise_equals_roundrobin(precision):
    hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=20, seed=3, precision=precision)
    a = lp.build_resnet_modules(lp.ResNetSpec(**SMALL), 3, 1, 2, hyper)
    b = lp.build_resnet_modules(lp.ResNetSpec(**SMALL), 3, 1, 2, hyper)
    rng = np.random.default_rng(5)
    data = [(rng.standard_normal((6, 8, 8, 3)), rng.integers(0, 5, 6)) for _ in range(6)]
    ma = lp.run_epoch(lp.RunMode.PPLL, a, iter(data), lp.RunConfig(buffer_capacity=2))
    mb = lp.run_deterministic(lp.RunMode.PPLL, b, iter(data), lp.RunConfig(buffer_capacity=2))
    assert ma.loss_history == mb.loss_history
    for x, z in zip(a, b):
        assert np.array_equal(_flat(x), _flat(z))


@pytest.mark.parametrize("N,H,Cin,Cout", [(4, 32, 16, 16), (2, 16, 32, 32), (4, 8, 64, 64),
                                          (2, 16, 16, 32), (6, 8, 64, 32), (128, 32, 16, 16),
                                          (128, 16, 32, 32), (128, 8, 64, 64), (16, 8, 32, 64),
                                          (4, 32, 32, 16), (2, 16, 32, 64)])
def test_implicit_conv3x3_wgrad_matches_torch(N, H, Cin, Cout):
    """The implicit-GEMM weight gradient (TMA tap windows read MN-major, taps
    stacked along M — or, for chunks of whole rows at Cin <= 32 and W >= 16, the
    halo form: three shifted copies, taps one image row apart — split-K
    partials reduced in fixed order) against the
    float64 torch weight gradient of conv2d on the same bf16 values, in the
    GEMM weight layout [9·Cin, Cout]; deterministic across runs.  Includes the
    ResNet-32 bench geometries at batch 128."""
    import torch.nn.functional as Fn
    from paper_2411_12780_b200 import _native as N_
    g = torch.Generator(device="cuda").manual_seed(7 * N + H + Cin)
    x = torch.randn(N, H, H, Cin, device="cuda", generator=g).bfloat16()
    dz = torch.randn(N, H, H, Cout, device="cuda", generator=g).bfloat16()
    lib = N_.load()
    s = torch.cuda.current_stream().cuda_stream
    nws = lib.ppll_conv3x3_wgrad_ws_floats(N, H, H, Cin, Cout)
    ws = torch.empty(nws, device="cuda")
    xr = x.double().permute(0, 3, 1, 2)
    wt = torch.zeros(Cout, Cin, 3, 3, dtype=torch.float64, device="cuda", requires_grad=True)
    y = Fn.conv2d(xr, wt, padding=1)
    y.backward(dz.double().permute(0, 3, 1, 2))
    # [Cout, Cin, 3, 3] -> GEMM layout [(3r+s)·Cin + ci, co]
    ref = wt.grad.permute(2, 3, 1, 0).reshape(9 * Cin, Cout)
    # exclusive GPU: the wide split-K form; shared GPU: one cluster with the
    # DSMEM reduction in-kernel
    # PPLL_CONV_WGRAD_HALO: 0 tap windows, 2 halo copies wherever the shape allows
    # (the default, 1, picks per form); read by the library on every call
    old_env = os.environ.get("PPLL_CONV_WGRAD_HALO")
    try:
        for halo in ("0", "2"):
            os.environ["PPLL_CONV_WGRAD_HALO"] = halo
            for exclusive in (1, 0):
                prev = lib.ppll_set_gpu_exclusive(exclusive)
                try:
                    outs = []
                    for _ in range(2):
                        dw = torch.full((9 * Cin, Cout), float("nan"), device="cuda")
                        N_.check(lib.ppll_conv3x3_wgrad_bf16(N, H, H, Cin, Cout, x.data_ptr(),
                                                             dz.data_ptr(), dw.data_ptr(),
                                                             ws.data_ptr(), nws, s), "conv wgrad")
                        torch.cuda.synchronize()
                        outs.append(dw.clone())
                finally:
                    lib.ppll_set_gpu_exclusive(prev)
                assert torch.equal(outs[0], outs[1]), (halo, exclusive)
                err = (outs[0].double() - ref).abs().max().item() / (ref.abs().max().item() + 1e-12)
                assert err < 1e-4, (halo, exclusive, err)
    finally:
        if old_env is None:
            os.environ.pop("PPLL_CONV_WGRAD_HALO", None)
        else:
            os.environ["PPLL_CONV_WGRAD_HALO"] = old_env


@pytest.mark.parametrize("N,H,Cin,Cout", [(4, 32, 16, 16), (2, 16, 32, 32), (4, 8, 64, 64),
                                          (2, 16, 16, 32), (6, 8, 64, 32)])
def test_implicit_conv3x3_matches_torch(N, H, Cin, Cout):
    """The implicit-GEMM conv (TMA 4-D window gathers, SW32/64/128 K-major
    tiles) against torch conv2d on the same bf16 values: forward and the
    transposed-convolution input gradient."""
    import torch.nn.functional as Fn
    from paper_2411_12780_b200 import _native as N_
    g = torch.Generator(device="cuda").manual_seed(N * H + Cin)
    x = torch.randn(N, H, H, Cin, device="cuda", generator=g).bfloat16()
    w = (torch.randn(9 * Cin, Cout, device="cuda", generator=g) / (9 * Cin) ** 0.5).bfloat16()
    dz = torch.randn(N, H, H, Cout, device="cuda", generator=g).bfloat16()
    lib = N_.load()
    s = torch.cuda.current_stream().cuda_stream
    y = torch.empty(N, H, H, Cout, device="cuda", dtype=torch.bfloat16)
    dx = torch.empty(N, H, H, Cin, device="cuda", dtype=torch.bfloat16)
    N_.check(lib.ppll_conv3x3_bf16(N, H, H, Cin, Cout, x.data_ptr(), w.data_ptr(), y.data_ptr(),
                                   0, s), "conv fwd")
    N_.check(lib.ppll_conv3x3_bf16(N, H, H, Cin, Cout, dz.data_ptr(), w.data_ptr(),
                                   dx.data_ptr(), 1, s), "conv dgrad")
    torch.cuda.synchronize()
    # torch weight [Cout, Cin, 3, 3] from the GEMM layout [(3r+s)·Cin + ci, co]
    wt = w.float().reshape(3, 3, Cin, Cout).permute(3, 2, 0, 1).contiguous()
    xr = x.float().permute(0, 3, 1, 2)
    ref = Fn.conv2d(xr, wt, padding=1).permute(0, 2, 3, 1)
    ref_dx = Fn.conv_transpose2d(dz.float().permute(0, 3, 1, 2), wt, padding=1).permute(0, 2, 3, 1)
    for got, want in ((y, ref), (dx, ref_dx)):
        err = (got.float() - want).abs().max().item() / (want.abs().max().item() + 1e-9)
        assert err < 1e-2, err
