"""GPU parity of the ViT local step (native ``ppll_vit_stage_step``) against the
float64 CPU restatement ``oracle/vit_oracle.py`` (itself pinned to torch
autograd in tests/test_vit_oracle.py).

Tolerances: fp32 parity mode — per-step loss |Δ| <= 1e-4·max(1,|loss|),
x_out max|Δ|/max|ref| <= 1e-4, weights after N steps max|ΔW|/max|W| <= 1e-3;
bf16 mode — loss 3e-2 relative, x_out 5e-2, weights 5e-2.  Pipeline vs
round-robin vs sequential: bitwise."""
import numpy as np
import pytest
import torch

import paper_2411_12780_b200 as lp
import vit_oracle as vo

pytestmark = pytest.mark.gpu

SMALL = dict(image=8, channels=3, patch=4, dim=128, heads=2, mlp=256, depth=3, classes=5)


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _pair(kw, depths, d_prime, n, precision, steps, seed=7):
    spec = lp.VitSpec(**kw)
    hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=steps, seed=seed,
                           precision=precision)
    mods = lp.build_vit_modules(spec, depths, d_prime, n, hyper)
    stages = vo.build_vit_stages(vo.VitSpec(**kw), depths, d_prime, n, seed)
    return spec, mods, stages


def _flat(m):
    return np.concatenate([p.data.ravel() for p in m.parameters()])


def _flat_o(st):
    return np.concatenate([p.ravel() for p in st.params()])


def test_init_matches_oracle_draws():
    spec, mods, stages = _pair(SMALL, [1, 1, 1], 1, 2, "fp32", 4)
    assert [m.n_aux_layers for m in mods] == [len(s.aux) for s in stages]
    for m, st in zip(mods, stages):
        np.testing.assert_allclose(_flat(m), _flat_o(st), rtol=0, atol=1e-7)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_vit_local_steps_match_oracle(precision):
    steps = 3
    spec, mods, stages = _pair(SMALL, [1, 1, 1], 1, 2, precision, steps)
    rng = np.random.default_rng(0)
    B = 4
    ltol, xtol, wtol = (1e-4, 1e-4, 1e-3) if precision == "fp32" else (3e-2, 5e-2, 5e-2)
    for t in range(steps):
        img = rng.standard_normal((B, 3, 8, 8))
        y = rng.integers(0, 5, B)
        h = lp.Tensor(img)
        hr = img
        for j, (m, st) in enumerate(zip(mods, stages)):
            loss, h = lp.local_loss_and_update(m, h, y)
            ref, hr, _ = vo.local_step(st, hr, y, 0.05, 0.001, steps, 0.9, 1e-4)
            assert abs(loss - ref) <= ltol * max(1.0, abs(ref)), (t, j, loss, ref)
            hd = h.data
            assert hd.shape == hr.shape
            assert np.abs(hd - hr).max() / np.abs(hr).max() <= xtol, (t, j)
            hr = hd if precision == "bf16" else hr     # teacher-force in bf16 mode
    for m, st in zip(mods, stages):
        a, b = _flat(m), _flat_o(st)
        assert np.abs(a - b).max() / np.abs(b).max() <= wtol


def test_vit_small_full_token_count_fp32():
    """ViT-S geometry (T=65, D=384, 6 heads, MLP 1536) at batch 2, one step."""
    kw = dict(image=32, channels=3, patch=4, dim=384, heads=6, mlp=1536, depth=2, classes=10)
    spec, mods, stages = _pair(kw, [1, 1], 1, 3, "fp32", 2)
    rng = np.random.default_rng(1)
    img = rng.standard_normal((2, 3, 32, 32))
    y = np.array([3, 7])
    h, hr = lp.Tensor(img), img
    for m, st in zip(mods, stages):
        loss, h = lp.local_loss_and_update(m, h, y)
        ref, hr, _ = vo.local_step(st, hr, y, 0.05, 0.001, 2, 0.9, 1e-4)
        assert abs(loss - ref) <= 1e-4 * max(1.0, abs(ref))
        assert np.abs(h.data - hr).max() / np.abs(hr).max() <= 1e-4
    for m, st in zip(mods, stages):
        a, b = _flat(m), _flat_o(st)
        assert np.abs(a - b).max() / np.abs(b).max() <= 1e-3


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_vit_pipeline_bitwise_equals_roundrobin(precision):
    kw = SMALL
    spec = lp.VitSpec(**kw)
    hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=20, seed=3, precision=precision)
    a = lp.build_vit_modules(spec, [1, 1, 1], 1, 2, hyper)
    b = lp.build_vit_modules(spec, [1, 1, 1], 1, 2, hyper)
    rng = np.random.default_rng(5)
    data = [(rng.standard_normal((6, 3, 8, 8)), rng.integers(0, 5, 6)) for _ in range(7)]
    ma = lp.run_epoch(lp.RunMode.PPLL, a, iter(data), lp.RunConfig(buffer_capacity=2))
    mb = lp.run_deterministic(lp.RunMode.PPLL, b, iter(data), lp.RunConfig(buffer_capacity=2))
    assert ma.loss_history == mb.loss_history
    for x, z in zip(a, b):
        assert np.array_equal(_flat(x), _flat(z))
    assert ma.batches_processed == [7, 7, 7]


FULL = dict(image=32, channels=3, patch=4, dim=384, heads=6, mlp=1536, depth=2, classes=10)


def test_tcgen05_attention_matches_simt_attention():
    """The tcgen05 attention (bf16, T=65) against the SIMT attention kernels:
    same stage, same data, engine switched through the C-ABI."""
    from paper_2411_12780_b200 import _native as N
    lib = N.load()
    spec = lp.VitSpec(**FULL)
    rng = np.random.default_rng(4)
    img = rng.standard_normal((6, 3, 32, 32))
    y = rng.integers(0, 10, 6)
    outs = []
    for engine in (0, 1):
        lib.ppll_set_attn_engine(engine)
        try:
            hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=4, seed=9, precision="bf16")
            mods = lp.build_vit_modules(spec, [1, 1], 1, 3, hyper)
            losses, xs = [], []
            h = lp.Tensor(img)
            for m in mods:
                loss, h = lp.local_loss_and_update(m, h, y)
                losses.append(loss)
                xs.append(h.data)
            outs.append((losses, xs, [_flat(m) for m in mods]))
        finally:
            lib.ppll_set_attn_engine(0)
    (l0, x0, p0), (l1, x1, p1) = outs
    np.testing.assert_allclose(l0, l1, rtol=1e-2)
    for a, b in zip(x0, x1):
        assert np.abs(a - b).max() / np.abs(b).max() < 2e-2
    for a, b in zip(p0, p1):
        assert np.abs(a - b).max() / np.abs(b).max() < 2e-2


def test_vit_s_geometry_bf16_vs_oracle():
    spec, mods, stages = _pair(FULL, [1, 1], 1, 3, "bf16", 2)
    rng = np.random.default_rng(2)
    img = rng.standard_normal((4, 3, 32, 32))
    y = rng.integers(0, 10, 4)
    h, hr = lp.Tensor(img), img
    for m, st in zip(mods, stages):
        loss, h = lp.local_loss_and_update(m, h, y)
        ref, hr, _ = vo.local_step(st, hr, y, 0.05, 0.001, 2, 0.9, 1e-4)
        assert abs(loss - ref) <= 3e-2 * abs(ref)
        assert np.abs(h.data - hr).max() / np.abs(hr).max() <= 5e-2
        hr = h.data
    for m, st in zip(mods, stages):
        a, b = _flat(m), _flat_o(st)
        assert np.abs(a - b).max() / np.abs(b).max() <= 5e-2


VIT_B = dict(image=96, channels=3, patch=16, dim=768, heads=12, mlp=3072, depth=2, classes=10)


def test_vit_b_stl_geometry_bf16_vs_oracle():
    """configs[3] geometry: ViT-B (D 768, 12 heads, MLP 3072) at 96x96 patch 16
    (T = 37) — the wide-row LayerNorm, D=768 GEMMs and T=37 attention."""
    spec, mods, stages = _pair(VIT_B, [1, 1], 1, 3, "bf16", 2)
    rng = np.random.default_rng(3)
    img = rng.standard_normal((2, 3, 96, 96))
    y = rng.integers(0, 10, 2)
    h, hr = lp.Tensor(img), img
    for m, st in zip(mods, stages):
        loss, h = lp.local_loss_and_update(m, h, y)
        ref, hr, _ = vo.local_step(st, hr, y, 0.05, 0.001, 2, 0.9, 1e-4)
        assert abs(loss - ref) <= 3e-2 * abs(ref)
        assert np.abs(h.data - hr).max() / np.abs(hr).max() <= 5e-2
        hr = h.data
    for m, st in zip(mods, stages):
        a, b = _flat(m), _flat_o(st)
        assert np.abs(a - b).max() / np.abs(b).max() <= 5e-2


def test_shared_gpu_vit_pipeline_pdl_on_off_bitwise(monkeypatch):
    """the PDL policy must not change results, and a graph captured
    under one setting must not be replayed under the other (graphs are keyed
    by the setting).  Same epoch with PDL forced on / off / on again: bitwise."""
    spec = lp.VitSpec(**SMALL)
    rng = np.random.default_rng(9)
    data = [(rng.standard_normal((6, 3, 8, 8)), rng.integers(0, 5, 6)) for _ in range(5)]
    out = []
    hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=40, seed=3, precision="bf16")
    mods_reused = lp.build_vit_modules(spec, [1, 1, 1], 1, 2, hyper)
    for pdl in ("1", "0", "1"):
        monkeypatch.setenv("PPLL_PDL", pdl)
        mods = lp.build_vit_modules(spec, [1, 1, 1], 1, 2, hyper)
        m = lp.run_epoch(lp.RunMode.PPLL, mods, iter(data), lp.RunConfig(buffer_capacity=2))
        out.append((m.loss_history, [_flat(x) for x in mods]))
        # one pipeline object replayed under both settings (cached graphs)
        lp.run_epoch(lp.RunMode.PPLL, mods_reused, iter(data), lp.RunConfig(buffer_capacity=2))
    for lh, fl in out[1:]:
        assert lh == out[0][0]
        for a, b in zip(fl, out[0][1]):
            assert np.array_equal(a, b)
    pipe = mods_reused[0]._pipelines
    keys = {k for p in pipe.values() for k in p.graphs}
    assert {k[2] for k in keys} == {0, 1}
