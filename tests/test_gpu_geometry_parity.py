"""Parity at the BENCHMARKED geometry (VERDICT r1 "What's weak" 1-2).

The bf16 stage steps of the bench workloads — ViT-S/4 (configs[1]: patch 4,
D 384, 6 heads, MLP 1536, T = 65, batch 128, cost split [1, 2, 2, 3], d'=1)
and ResNet-32/4 (configs[0]: 32x32, batch 128, cost split, implicit-GEMM
convolutions) — run for 5 steps through the public ``local_loss_and_update``
and are compared with the float64 restatement (oracle/torch_cpu.py, pinned to
the numpy oracles by tests/test_torch_cpu.py) on the same init and inputs.
Every stage is teacher-forced: its oracle input is the device's own x_out of
the previous stage, so each stage's error is its own.

What is compared (SURVEY §8c asks for loss / x_out / weights; round 1's
``max|W_dev - W_ref| / max|W|`` bar could not tell a stepped stage from an
unstepped one, because 3 steps move the weights by only ~4 % of max|W|):

* the UPDATE: dθ = θ_5 - θ_0 of the device vs the oracle, per parameter
  tensor, as ||dθ_dev - dθ_ref||_2 / ||dθ_ref||_2 — a stage that never
  stepped scores 1.0, a sign error 2.0; the bar is DTHETA_TOL for the whole
  stage and DTHETA_TENSOR_TOL for every tensor that moved;
* the per-step loss, relative (LOSS_TOL);
* x_out (the pushed boundary activation), max-abs error over max|ref| (XOUT_TOL).

Tolerances: bf16 tensor-core operands (8-bit mantissa, 2^-9 relative
rounding) with fp32 accumulation, bf16-stored activations.  ViT: the bars are
~3x the errors measured on a B200 (profiles/r02_geometry_parity.json: loss
2e-3, x_out 1.1e-2, dθ 0.7 % per stage).  ResNet: train-mode BatchNorm makes
bf16 rounding grow with depth (the 12-conv final stage's dθ is ~11 % off the
float64 update, the BN γ/β updates 20-25 %), so the bar is the bf16 NOISE
FLOOR itself: the same 5 steps in torch-CPU with bf16 autocast (convs in bf16,
BN/loss/update in fp32) give the same errors against float64, and the device
must stay within 1.3x of that floor (+0.01) on every stage.
"""
import copy
import json
import os

import numpy as np
import pytest
import torch

import paper_2411_12780_b200 as lp
import resnet_oracle as ro
import torch_cpu as tc
import vit_oracle as vo

pytestmark = pytest.mark.gpu

STEPS = 5
HP = dict(lr0=0.05, lr_min=0.001)
LOSS_TOL = 6e-3
XOUT_TOL = 3e-2
DTHETA_TOL = 2.5e-2
DTHETA_TENSOR_TOL = 4e-2
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    torch.set_num_threads(max(1, len(os.sched_getaffinity(0))))


def _dev_params(m):
    return [p.data.astype(np.float64).copy() for p in m.parameters()]


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _run(mods, tstages, xs, ys, tag, emulated=None, tol=None):
    """5 teacher-forced bf16 steps; returns the measured error summary.
    ``emulated``: fp32 TorchStages stepped under bf16 autocast on the same
    inputs (the bf16 noise floor, see the module docstring)."""
    tol = tol or {}
    th0_dev = [_dev_params(m) for m in mods]
    th0_ref = [[p.detach().numpy().copy() for p in ts.params] for ts in tstages]
    for a, b in zip(th0_dev, th0_ref):               # same init (fp32 rounding)
        for x, z in zip(a, b):
            assert x.shape == z.shape
            np.testing.assert_allclose(x, z, rtol=0, atol=1e-6 * max(1.0, np.abs(z).max()))
    rep = {"loss_rel": [], "xout_rel": [], "dtheta_stage": [], "dtheta_worst_tensor": []}
    for t in range(STEPS):
        h = lp.Tensor(xs[t])
        for j, (m, ts) in enumerate(zip(mods, tstages)):
            x_ref = xs[t] if j == 0 else h_prev
            loss, h = lp.local_loss_and_update(m, h, ys[t])
            ref, hr, _ = tc.local_step(ts, torch.as_tensor(x_ref, dtype=torch.float64), ys[t],
                                       HP["lr0"], HP["lr_min"], STEPS, 0.9, 1e-4)
            if emulated is not None:
                with torch.autocast("cpu", dtype=torch.bfloat16):
                    tc.local_step(emulated[j], torch.as_tensor(x_ref, dtype=torch.float32), ys[t],
                                  HP["lr0"], HP["lr_min"], STEPS, 0.9, 1e-4)
            hd = h.data.astype(np.float64)
            rep["loss_rel"].append(abs(loss - ref) / abs(ref))
            rep["xout_rel"].append(float(np.abs(hd - hr.numpy()).max() / np.abs(hr.numpy()).max()))
            h_prev = hd                              # teacher forcing: device x_out
    for j, (m, ts) in enumerate(zip(mods, tstages)):
        d_dev = [b - a for a, b in zip(th0_dev[j], _dev_params(m))]
        d_ref = [p.detach().numpy() - a for a, p in zip(th0_ref[j], ts.params)]
        cat = lambda L: np.concatenate([x.ravel() for x in L])  # noqa: E731
        rep["dtheta_stage"].append(_rel(cat(d_dev), cat(d_ref)))
        if emulated is not None:
            d_emu = [p.detach().double().numpy() - a for a, p in zip(th0_ref[j], emulated[j].params)]
            rep.setdefault("dtheta_bf16_floor", []).append(_rel(cat(d_emu), cat(d_ref)))
        moved = [(_rel(a, b), np.linalg.norm(b)) for a, b in zip(d_dev, d_ref)]
        big = max(n for _, n in moved)
        rep["dtheta_worst_tensor"].append(max(r for r, n in moved if n > 1e-3 * big))
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, "geometry_parity.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[tag] = {k: (max(v) if v else None) for k, v in rep.items()} | {"per_stage": rep}
    json.dump(data, open(path, "w"), indent=1)
    assert max(rep["loss_rel"]) <= tol.get("loss", LOSS_TOL), rep["loss_rel"]
    assert max(rep["xout_rel"]) <= tol.get("xout", XOUT_TOL), rep["xout_rel"]
    assert max(rep["dtheta_stage"]) <= tol.get("dtheta", DTHETA_TOL), rep["dtheta_stage"]
    assert max(rep["dtheta_worst_tensor"]) <= tol.get("tensor", DTHETA_TENSOR_TOL), \
        rep["dtheta_worst_tensor"]
    s = len(mods)
    if "first_loss" in tol:        # step 0: same parameters on both sides
        assert max(rep["loss_rel"][:s]) <= tol["first_loss"], rep["loss_rel"][:s]
        assert max(rep["xout_rel"][:s]) <= tol["first_xout"], rep["xout_rel"][:s]
    if emulated is not None:
        for got, floor in zip(rep["dtheta_stage"], rep["dtheta_bf16_floor"]):
            assert got <= 1.3 * floor + 0.01, (rep["dtheta_stage"], rep["dtheta_bf16_floor"])
    # the update is real: every stage moved and the check would catch "no step"
    assert all(r < 0.5 for r in rep["dtheta_stage"])


def test_vit_s_bench_config_bf16_update_parity():
    kw = dict(image=32, channels=3, patch=4, dim=384, heads=6, mlp=1536, depth=8, classes=10)
    spec = lp.VitSpec(**kw)
    depths = lp.balanced_vit_depths(spec, 4, 1, 3)
    assert depths == [1, 2, 2, 3]
    hyper = lp.Hyperparams(total_steps=STEPS, seed=42, precision="bf16", **HP)
    mods = lp.build_vit_modules(spec, depths, 1, 3, hyper)
    stages = vo.build_vit_stages(vo.VitSpec(**kw), depths, 1, 3, 42)
    tst = [tc.from_vit(s, torch.float64) for s in stages]
    rng = np.random.default_rng(11)
    B = 128
    xs = rng.standard_normal((STEPS, B, 3, 32, 32)).astype(np.float32)
    ys = rng.integers(0, 10, (STEPS, B))
    _run(mods, tst, xs, ys, "vit_s_b128_bf16")


def test_resnet32_bench_config_bf16_update_parity():
    from paper_2411_12780_b200.resnet import balanced_resnet_split
    kw = dict(n=5, image=32, channels=3, widths=(16, 32, 64), classes=10)
    spec = lp.ResNetSpec(**kw)
    split = balanced_resnet_split(spec, 4, 1, 3)
    hyper = lp.Hyperparams(total_steps=STEPS, seed=42, precision="bf16", **HP)
    mods = lp.build_resnet_modules(spec, 4, 1, 3, hyper, split=split)
    stages = ro.build_resnet_stages(ro.ResNetSpec(**kw), 4, 1, 3, 42, split=split)
    tst = [tc.from_resnet(copy.deepcopy(s), torch.float64) for s in stages]
    emu = [tc.from_resnet(copy.deepcopy(s), torch.float32) for s in stages]
    rng = np.random.default_rng(12)
    B = 128
    xs = rng.standard_normal((STEPS, B, 32, 32, 3)).astype(np.float32)
    ys = rng.integers(0, 10, (STEPS, B))
    _run(mods, tst, xs, ys, "resnet32_b128_bf16", emulated=emu,
         tol={"loss": 2e-3, "xout": 6e-2, "dtheta": 0.15, "tensor": 0.35})


@pytest.mark.parametrize("C", [16, 32, 64])
def test_transposed_conv_epilogue_32x32(C):
    """The basic block's input-gradient convolution with its fused epilogue
    (resnet_stage.cu conv_bn_bwd): dx = (convT(dz, W) + dres) * [a > 0] at
    32x32, batch 128 — through the C-ABI ``ppll_conv3x3_bf16_ex``."""
    import torch.nn.functional as Fn
    from paper_2411_12780_b200 import _native as N_
    g = torch.Generator(device="cuda").manual_seed(C)
    B, H = 128, 32
    w = (torch.randn(9 * C, C, device="cuda", generator=g) / (9 * C) ** 0.5).bfloat16()
    dz = torch.randn(B, H, H, C, device="cuda", generator=g).bfloat16()
    dres = torch.randn(B, H, H, C, device="cuda", generator=g).bfloat16()
    act = torch.relu(torch.randn(B, H, H, C, device="cuda", generator=g)).bfloat16()
    act[0, 0, 0, :] = 0.0                             # ReLU'(0) = 0 (tensor.py:156)
    dx = torch.empty_like(dz)
    lib = N_.load()
    N_.check(lib.ppll_conv3x3_bf16_ex(B, H, H, C, C, dz.data_ptr(), w.data_ptr(), dx.data_ptr(),
                                      1, dres.data_ptr(), act.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream), "convT epilogue")
    torch.cuda.synchronize()
    wt = w.double().reshape(3, 3, C, C).permute(3, 2, 0, 1)
    ref = Fn.conv_transpose2d(dz.double().permute(0, 3, 1, 2), wt, padding=1).permute(0, 2, 3, 1)
    ref = (ref + dres.double()) * (act.double() > 0)
    got = dx.double()
    assert torch.all(got[act == 0] == 0)
    err = ((got - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-2, err
    # forward with residual and mask too
    y = torch.empty_like(dz)
    N_.check(lib.ppll_conv3x3_bf16_ex(B, H, H, C, C, dz.data_ptr(), w.data_ptr(), y.data_ptr(),
                                      0, dres.data_ptr(), act.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream), "conv epilogue")
    torch.cuda.synchronize()
    ref = Fn.conv2d(dz.double().permute(0, 3, 1, 2), wt, padding=1).permute(0, 2, 3, 1)
    ref = (ref + dres.double()) * (act.double() > 0)
    err = ((y.double() - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-2, err


# --------------------------------------------------------------------------
# a8: the non-finite guard on the device path (tensor.py:41-43)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("family", ["mlp", "vit", "resnet"])
def test_nan_input_raises_nonfinite_and_skips_update(family):
    if family == "mlp":
        spec = lp.NetworkSpec((48, 32, 32, 10))
        hyper = lp.Hyperparams(total_steps=4, seed=1, precision="bf16")
        mods = lp.build_modules(spec, lp.partition(spec, 2), 1, 3, hyper)
        x = np.random.default_rng(0).standard_normal((8, 48))
    elif family == "vit":
        spec = lp.VitSpec(image=8, channels=3, patch=4, dim=128, heads=2, mlp=256, depth=2,
                          classes=10)
        hyper = lp.Hyperparams(total_steps=4, seed=1, precision="bf16")
        mods = lp.build_vit_modules(spec, [1, 1], 1, 3, hyper)
        x = np.random.default_rng(0).standard_normal((8, 3, 8, 8))
    else:
        spec = lp.ResNetSpec(n=1, image=8, channels=3, widths=(16, 32, 64), classes=10)
        hyper = lp.Hyperparams(total_steps=4, seed=1, precision="bf16")
        mods = lp.build_resnet_modules(spec, 2, 1, 3, hyper)
        x = np.random.default_rng(0).standard_normal((16, 8, 8, 3))
    y = np.arange(x.shape[0]) % 10
    m = mods[0]
    before = np.concatenate([p.data.ravel() for p in m.parameters()])
    bad = x.copy()
    bad.reshape(-1)[5] = np.nan
    with pytest.raises(lp.NonFiniteError):
        lp.local_loss_and_update(m, lp.Tensor(bad), y)
    assert m.optimizer.step_count == 0
    after = np.concatenate([p.data.ravel() for p in m.parameters()])
    assert np.array_equal(before, after)            # no partial update
    # the module is usable again; an Inf through the pipeline surfaces as
    # WorkerPanic(stage 0) from run_epoch (runtime.py:400-402)
    loss, _ = lp.local_loss_and_update(m, lp.Tensor(x), y)
    assert np.isfinite(loss)
    bad[...] = x
    bad.reshape(-1)[0] = np.inf
    with pytest.raises(lp.WorkerPanic) as ei:
        lp.run_epoch(lp.RunMode.PPLL, mods, iter([(x, y), (bad, y)]),
                     lp.RunConfig(buffer_capacity=2))
    assert ei.value.stage_index == 0


@pytest.mark.parametrize("family", ["vit", "resnet"])
def test_bench_config_fp32_update_parity(family):
    """The same 5 steps in the fp32 parity mode: with no bf16 rounding the
    device update matches the float64 one to fp32 precision at the full
    geometry — the algorithm (not just its bf16 noise) is the reference's."""
    rng = np.random.default_rng(13)
    hyper = lp.Hyperparams(total_steps=STEPS, seed=42, precision="fp32", **HP)
    if family == "vit":
        kw = dict(image=32, channels=3, patch=4, dim=384, heads=6, mlp=1536, depth=8, classes=10)
        depths = lp.balanced_vit_depths(lp.VitSpec(**kw), 4, 1, 3)
        mods = lp.build_vit_modules(lp.VitSpec(**kw), depths, 1, 3, hyper)
        tst = [tc.from_vit(s, torch.float64)
               for s in vo.build_vit_stages(vo.VitSpec(**kw), depths, 1, 3, 42)]
        xs = rng.standard_normal((STEPS, 128, 3, 32, 32)).astype(np.float32)
    else:
        from paper_2411_12780_b200.resnet import balanced_resnet_split
        kw = dict(n=5, image=32, channels=3, widths=(16, 32, 64), classes=10)
        split = balanced_resnet_split(lp.ResNetSpec(**kw), 4, 1, 3)
        mods = lp.build_resnet_modules(lp.ResNetSpec(**kw), 4, 1, 3, hyper, split=split)
        tst = [tc.from_resnet(s, torch.float64)
               for s in ro.build_resnet_stages(ro.ResNetSpec(**kw), 4, 1, 3, 42, split=split)]
        xs = rng.standard_normal((STEPS, 128, 32, 32, 3)).astype(np.float32)
    ys = rng.integers(0, 10, (STEPS, 128))
    # step 0 (identical parameters) agrees to fp32 rounding in both families.
    # ViT stays there for all 5 steps (dθ 4e-6 measured).  ResNet-32's deep
    # BN stage amplifies fp32 rounding step over step (stage 3 x_out error
    # 1e-6 -> 2e-4 -> 1e-3 -> 3e-3 over steps 0-4; dθ 1.4 %): a property of
    # the trajectory, not of one step, hence the looser multi-step bar.
    tol = ({"loss": 1e-6, "xout": 2e-5, "dtheta": 5e-5, "tensor": 2e-3} if family == "vit" else
           {"loss": 5e-5, "xout": 1e-2, "dtheta": 4e-2, "tensor": 0.1})
    _run(mods, tst, xs, ys, f"{family}_b128_fp32",
         tol=tol | {"first_loss": 1e-6, "first_xout": 3e-6})
