"""The paper's E2E and naive-PP baselines (reference runtime.py:248-284 E2E,
:359-382 NaivePP) for the ViT and ResNet families, on the device.

Checker: ``oracle/torch_cpu.e2e_step`` in float64 — autograd through the
chained stage blocks (the final stage's block ends in its task head), the
reference's Nesterov on the parameters on that path only — which
tests/test_torch_cpu.py pins to the reference's own E2E runs
(tests/golden/e2e_naive.npz, MLP) to 1e-12.

Per run: ``run_deterministic`` and ``run_epoch`` in E2E and NAIVE_PP modes
on fresh, identically initialised modules.  Tolerances: fp32 parity mode —
final-stage loss per batch |Δ| <= 2e-4·max(1,|loss|); the update
dθ = θ_N - θ_0 of every stage within 2e-3 (ViT) / 5e-3 (ResNet, train-mode
BN) of the float64 update in relative L2 norm; bf16 — loss 2e-2 relative, dθ
within 6e-2 (ViT); ResNet bf16 — train-mode BatchNorm over 16-256 pixels per
channel amplifies bf16 rounding as the gradient crosses three stages, so its
bar is the bf16 NOISE FLOOR: the same E2E steps in torch-CPU under bf16
autocast (convs in bf16) against float64, with the device within 1.3x of that
floor + 0.02 per stage (a stage that never stepped scores 1.0).
Aux-head parameters are bitwise untouched, step counters advance once per
batch, and the four device runs are bitwise identical to each other.
"""
import copy

import numpy as np
import pytest
import torch

import paper_2411_12780_b200 as lp
import resnet_oracle as ro
import torch_cpu as tc
import vit_oracle as vo

pytestmark = pytest.mark.gpu

HP = (0.05, 0.001)
VIT = dict(image=8, channels=3, patch=4, dim=128, heads=2, mlp=256, depth=3, classes=5)
RES = dict(n=1, image=8, channels=3, widths=(16, 32, 64), classes=5)
TOL = {("vit", "fp32"): (2e-4, 2e-3), ("vit", "bf16"): (2e-2, 6e-2),
       ("resnet", "fp32"): (2e-4, 5e-3), ("resnet", "bf16"): (2e-2, None)}


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _flat(m):
    return np.concatenate([p.data.astype(np.float64).ravel() for p in m.parameters()])


def _build(family, precision, steps):
    hyper = lp.Hyperparams(lr0=HP[0], lr_min=HP[1], total_steps=steps, seed=7,
                           precision=precision)
    if family == "vit":
        return lp.build_vit_modules(lp.VitSpec(**VIT), [1, 1, 1], 1, 2, hyper)
    return lp.build_resnet_modules(lp.ResNetSpec(**RES), 3, 1, 2, hyper)


def _oracle(family):
    if family == "vit":
        return [tc.from_vit(s, torch.float64)
                for s in vo.build_vit_stages(vo.VitSpec(**VIT), [1, 1, 1], 1, 2, 7)]
    return [tc.from_resnet(copy.deepcopy(s), torch.float64)
            for s in ro.build_resnet_stages(ro.ResNetSpec(**RES), 3, 1, 2, 7)]


def _data(family, steps, B=4):
    rng = np.random.default_rng(5)
    shape = (B, 3, 8, 8) if family == "vit" else (B, 8, 8, 3)
    return [(rng.standard_normal(shape).astype(np.float32), rng.integers(0, 5, B))
            for _ in range(steps)]


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("family", ["vit", "resnet"])
def test_e2e_and_naive_pp_match_autograd(family, precision):
    steps = 4
    data = _data(family, steps)
    ltol, dtol = TOL[(family, precision)]
    tst = _oracle(family)
    th0 = [np.concatenate([p.detach().numpy().ravel() for p in ts.params]) for ts in tst]
    ref_l = [tc.e2e_step(tst, x, y, HP[0], HP[1], steps, 0.9, 1e-4) for x, y in data]
    d_ref = [np.concatenate([p.detach().numpy().ravel() for p in ts.params]) - a
             for ts, a in zip(tst, th0)]
    floor = None
    if dtol is None:                    # ResNet bf16: the autocast noise floor
        emu = [tc.TorchStage(ts.index, [p.detach().float().numpy() for p in ts.params],
                             ts.block_fn, ts.head_fn, torch.float32) for ts in _oracle(family)]
        for x, y in data:
            with torch.autocast("cpu", dtype=torch.bfloat16):
                tc.e2e_step(emu, x, y, HP[0], HP[1], steps, 0.9, 1e-4)
        floor = [np.linalg.norm(np.concatenate([p.detach().double().numpy().ravel()
                                                for p in e.params]) - a - d) / np.linalg.norm(d)
                 for e, a, d in zip(emu, th0, d_ref)]
    runs = []
    for mode in (lp.RunMode.E2E, lp.RunMode.NAIVE_PP):
        for runner in (lp.run_deterministic, lp.run_epoch):
            mods = _build(family, precision, steps)
            init = [_flat(m) for m in mods]
            met = runner(mode, mods, iter(data), lp.RunConfig(buffer_capacity=2))
            runs.append((met, mods, init))
    s = len(runs[0][1])
    for met, mods, init in runs:
        assert met.n_batches == steps and met.batches_processed == [steps] * s
        got = np.array(met.loss_history[-1])
        ref = np.array(ref_l)
        if precision == "fp32":
            assert np.abs(got - ref).max() <= ltol * max(1.0, np.abs(ref).max()), (got, ref)
        else:
            assert (np.abs(got - ref) / np.abs(ref)).max() <= ltol, (got, ref)
        for j, m in enumerate(mods):
            np.testing.assert_allclose(init[j], th0[j], rtol=0, atol=1e-6)   # same init
            fin = _flat(m)
            d_dev = fin - init[j]
            rel = np.linalg.norm(d_dev - d_ref[j]) / np.linalg.norm(d_ref[j])
            bar = dtol if floor is None else 1.3 * floor[j] + 0.02
            assert rel <= bar and rel < 0.5, (j, rel, bar)
            # aux parameters (off the E2E path) are bitwise untouched
            nb = sum(p.data.size for p in m.block_parameters())
            if j < s - 1:
                assert nb < fin.size
                assert np.array_equal(fin[nb:], init[j][nb:])
            assert m.optimizer.step_count == steps == m.device_step()
    base = runs[0]
    for met, mods, _ in runs[1:]:
        assert met.loss_history == base[0].loss_history
        for a, b in zip(mods, base[1]):
            assert np.array_equal(_flat(a), _flat(b))


def test_e2e_is_not_local_learning():
    """E2E and PPLL differ (the boundary gradient reaches the earlier
    stages): after the same batches stage 0's parameters differ."""
    data = _data("vit", 2)
    a = _build("vit", "fp32", 2)
    b = _build("vit", "fp32", 2)
    lp.run_deterministic(lp.RunMode.E2E, a, iter(data), lp.RunConfig(buffer_capacity=2))
    lp.run_deterministic(lp.RunMode.PPLL, b, iter(data), lp.RunConfig(buffer_capacity=2))
    assert not np.array_equal(_flat(a[0]), _flat(b[0]))
