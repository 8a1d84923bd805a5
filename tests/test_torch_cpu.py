"""The torch-CPU restatement (oracle/torch_cpu.py, the ViT/ResNet CPU baseline
of BASELINE.md §3) against the float64 numpy oracles: autograd vs the manual
backward, same init, same step order — float64 to 1e-9, float32 to fp32
rounding."""
import copy

import numpy as np
import pytest
import torch

import ppll_oracle as orc
import resnet_oracle as ro
import torch_cpu as tc
import vit_oracle as vo

HP = (0.05, 0.001, 10, 0.9, 1e-4)


def _run(stages, tstages, xs, ys, steps):
    out = []
    for t in range(steps):
        h, ht = xs[t], xs[t]
        for st, ts in zip(stages, tstages):
            if isinstance(st, orc.OracleStage):
                lo, h, _ = orc.local_step(st, h, ys[t], *HP)
            elif isinstance(st, vo.VitStage):
                lo, h, _ = vo.local_step(st, h, ys[t], *HP)
            else:
                lo, h, _ = ro.local_step(st, h, ys[t], *HP)
            lt, ht, _ = tc.local_step(ts, ht, ys[t], *HP)
            out.append((lo, lt, h, ht.numpy()))
    return out


def _check(stages, tstages, rtol):
    for st, ts in zip(stages, tstages):
        for p, q in zip(st.params(), ts.params):
            q = q.detach().numpy()
            assert p.shape == q.shape
            assert np.max(np.abs(p - q)) <= rtol * max(1e-3, np.max(np.abs(p)))


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-9), (torch.float32, 2e-4)])
def test_vit_restatement(dtype, tol):
    spec = vo.VitSpec(image=8, channels=3, patch=4, dim=16, heads=2, mlp=32, depth=3, classes=5)
    stages = vo.build_vit_stages(spec, [2, 1], 2, 1, 42)
    tst = [tc.from_vit(copy.deepcopy(s), dtype) for s in stages]
    rng = np.random.default_rng(0)
    xs = rng.standard_normal((3, 4, 3, 8, 8))
    ys = rng.integers(0, 5, (3, 4))
    for lo, lt, h, ht in _run(stages, tst, xs, ys, 3):
        assert abs(lo - lt) <= tol * max(1.0, abs(lo))
        assert np.max(np.abs(h - ht)) <= tol * max(1.0, np.max(np.abs(h)))
    _check(stages, tst, tol)


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-9), (torch.float32, 5e-4)])
def test_resnet_restatement(dtype, tol):
    spec = ro.ResNetSpec(n=1, image=8, channels=3, widths=(4, 8, 8), classes=5)
    stages = ro.build_resnet_stages(spec, 2, 2, 1, 42, split=[[0, 1], [2]])
    tst = [tc.from_resnet(copy.deepcopy(s), dtype) for s in stages]
    rng = np.random.default_rng(1)
    xs = rng.standard_normal((3, 4, 8, 8, 3))
    ys = rng.integers(0, 5, (3, 4))
    for lo, lt, h, ht in _run(stages, tst, xs, ys, 3):
        assert abs(lo - lt) <= tol * max(1.0, abs(lo))
        assert np.max(np.abs(h - ht)) <= tol * max(1.0, np.max(np.abs(h)))
    _check(stages, tst, tol)


def test_mlp_restatement():
    dims = (12, 10, 9, 8, 5)
    stages = orc.build_stages(dims, orc.partition(dims, 2), 2, 3, 42)
    tst = [tc.from_mlp(copy.deepcopy(s), torch.float64) for s in stages]
    rng = np.random.default_rng(2)
    xs = rng.standard_normal((4, 6, 12))
    ys = rng.integers(0, 5, (4, 6))
    for lo, lt, h, ht in _run(stages, tst, xs, ys, 4):
        assert abs(lo - lt) <= 1e-12
        np.testing.assert_allclose(h, ht, rtol=0, atol=1e-12)
    _check(stages, tst, 1e-12)


def test_adamw_rule_matches_torch_optim_adamw():
    """oracle/torch_cpu.py's AdamW branch == torch.optim.AdamW step for step."""
    dims = (12, 10, 5)
    stages = orc.build_stages(dims, orc.partition(dims, 1), 1, 3, 42)
    ts = tc.from_mlp(copy.deepcopy(stages[0]), torch.float64)
    ref = [torch.tensor(p, requires_grad=True) for p in stages[0].params()]
    rng = np.random.default_rng(4)
    for t in range(4):
        x = rng.standard_normal((6, 12))
        y = rng.integers(0, 5, 6)
        lr = tc.cosine_lr(t, 0.05, 0.001, 10)
        tc.local_step(ts, x, y, 0.05, 0.001, 10, 0.9, 1e-2, opt="adamw")
        opt = torch.optim.AdamW(ref, lr=lr, betas=(0.9, 0.999), eps=1e-8, weight_decay=1e-2)
        if t:
            opt.load_state_dict(state)
            for gr in opt.param_groups:
                gr["lr"] = lr
        h = torch.tensor(x)
        for i, (W, b) in enumerate(zip(ref[0::2], ref[1::2])):
            h = h @ W + b
            if i < len(ref) // 2 - 1:
                h = torch.relu(h)
        loss = torch.nn.functional.cross_entropy(h, torch.tensor(y))
        opt.zero_grad()
        loss.backward()
        opt.step()
        state = opt.state_dict()
    for p, q in zip(ts.params, ref):
        np.testing.assert_allclose(p.detach().numpy(), q.detach().numpy(), rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("tag", ["s2", "s4", "s3"])
def test_e2e_step_matches_reference_e2e(tag):
    """tc.e2e_step (autograd through the chained blocks) against the
    reference's own E2E / naive-PP runs (tests/golden/e2e_naive.npz, generated
    by importing the reference): this pins the checker the ViT / ResNet E2E
    GPU tests use."""
    import os
    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "e2e_naive.npz"))
    dims = tuple(int(d) for d in z[f"{tag}_dims"])
    s = int(z[f"{tag}_s"])
    stages = orc.build_stages(dims, orc.partition(dims, s), 2, 3, 42)
    tst = [tc.from_mlp(copy.deepcopy(st), torch.float64) for st in stages]
    losses = [tc.e2e_step(tst, x, y, 0.05, 0.001, 10, 0.9, 1e-4)
              for x, y in zip(z[f"{tag}_xs"], z[f"{tag}_ys"])]
    np.testing.assert_allclose(losses, z[f"{tag}_losses"], rtol=0, atol=1e-12)
    for j, ts in enumerate(tst):
        f = np.concatenate([p.detach().numpy().ravel() for p in ts.params])
        np.testing.assert_allclose(f, z[f"{tag}_final_{j}"], rtol=0, atol=1e-12)
        assert ts.step_count == int(z[f"{tag}_step_{j}"])


def test_e2e_step_vit_resnet_leave_aux_untouched():
    """E2E through ViT / ResNet stages: aux parameters never move, block
    parameters do."""
    vspec = vo.VitSpec(image=8, channels=3, patch=4, dim=128, heads=2, mlp=256, depth=3, classes=5)
    rspec = ro.ResNetSpec(n=1, image=8, channels=3, widths=(16, 32, 64), classes=5)
    cases = [([tc.from_vit(s) for s in vo.build_vit_stages(vspec, [1, 1, 1], 1, 2, 7)],
              np.random.default_rng(0).standard_normal((4, 3, 8, 8))),
             ([tc.from_resnet(s) for s in ro.build_resnet_stages(rspec, 3, 1, 2, 7)],
              np.random.default_rng(0).standard_normal((4, 8, 8, 3)))]
    for tst, x in cases:
        before = [[p.detach().clone() for p in ts.params] for ts in tst]
        tc.e2e_step(tst, x, np.array([0, 1, 2, 3]), 0.05, 0.001, 4, 0.9, 1e-4)
        for j, ts in enumerate(tst):
            moved = [not torch.equal(a, b) for a, b in zip(before[j], ts.params)]
            assert any(moved)
            if j < len(tst) - 1:
                assert not all(moved)          # aux head parameters are untouched
