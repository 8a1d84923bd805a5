"""Pin the ViT oracle's manual backward against torch.autograd (float64, CPU).

There is no reference implementation of ViT blocks; this test is
what makes the restatement trustworthy: an independent autograd derivation of
the same forward must give the same gradients, and the step must follow the
reference's update semantics (cosine LR, L2-in-gradient Nesterov on every
parameter)."""
import math

import numpy as np
import pytest
import torch

import vit_oracle as vo
from ppll_oracle import cosine_lr, nesterov_update

SPEC = vo.VitSpec(image=8, channels=3, patch=4, dim=16, heads=2, mlp=32, depth=3, classes=5)


def _torch_forward(st, x_in, y):
    """Same math as vit_oracle, written with torch ops; returns (loss, params)."""
    spec = st.spec
    names = st.param_list()
    P = [torch.tensor(a, dtype=torch.float64, requires_grad=True) for _, _, a in names]
    it = iter(P)
    x = torch.tensor(x_in, dtype=torch.float64)

    def ln(t, g, b):
        return torch.nn.functional.layer_norm(t, (t.shape[-1],), g, b, eps=vo.LN_EPS)

    if st.patch is not None:
        wpe, bpe, cls, pos = next(it), next(it), next(it), next(it)
        B = x.shape[0]
        p = spec.patch
        pt = x.reshape(B, spec.channels, spec.image // p, p, spec.image // p, p)
        pt = pt.permute(0, 2, 4, 1, 3, 5).reshape(B, spec.n_patches, spec.patch_dim)
        tok = pt @ wpe + bpe
        x = torch.cat([cls.expand(B, 1, spec.dim), tok], 1) + pos

    def layer(x):
        g1, b1_, wqkv, bqkv, wo, bo, g2, b2_, w1, b1, w2, b2 = [next(it) for _ in range(12)]
        B, T, D = x.shape
        H, dh = spec.heads, D // spec.heads
        qkv = ln(x, g1, b1_) @ wqkv + bqkv
        q, k, v = [qkv[..., i * D:(i + 1) * D].reshape(B, T, H, dh).transpose(1, 2)
                   for i in range(3)]
        a = torch.softmax(q @ k.transpose(-1, -2) / math.sqrt(dh), -1) @ v
        x1 = x + a.transpose(1, 2).reshape(B, T, D) @ wo + bo
        u = ln(x1, g2, b2_) @ w1 + b1
        return x1 + torch.nn.functional.gelu(u) @ w2 + b2

    for _ in st.block:
        x = layer(x.detach() if False else x)
    for _ in st.aux:
        x = layer(x)
    lg, lb, wh, bh = next(it), next(it), next(it), next(it)
    logits = ln(x[:, 0], lg, lb) @ wh + bh
    loss = torch.nn.functional.cross_entropy(logits, torch.tensor(y))
    return loss, P


@pytest.mark.parametrize("j", [0, 1, 2])
def test_manual_backward_matches_autograd(j):
    stages = vo.build_vit_stages(SPEC, [1, 1, 1], d_prime=2, n=2, seed=7)
    st = stages[j]
    rng = np.random.default_rng(j)
    B = 3
    if j == 0:
        x = rng.standard_normal((B, SPEC.channels, SPEC.image, SPEC.image))
    else:
        x = rng.standard_normal((B, SPEC.tokens, SPEC.dim))
    y = rng.integers(0, SPEC.classes, B)
    loss, x_out, logits, grads = vo.local_grads(st, x, y)
    tl, P = _torch_forward(st, x, y)
    tl.backward()
    assert abs(loss - tl.item()) < 1e-12
    names = st.param_list()
    assert len(grads) == len(P) == len(names)
    for (grp, key, _), g, p in zip(names, grads, P):
        np.testing.assert_allclose(g, p.grad.numpy(), rtol=1e-9, atol=1e-11,
                                   err_msg=f"{grp}.{key}")


def test_structure_and_init_order():
    stages = vo.build_vit_stages(vo.VitSpec(), [2, 2, 2, 2], d_prime=1, n=3, seed=42)
    assert [len(s.aux) for s in stages] == [1, 1, 1, 0]      # aux_depth(l,1,3); none on final
    assert stages[0].patch is not None and stages[1].patch is None
    assert [s.final for s in stages] == [False, False, False, True]
    # per-stage seeds: a stage's init does not depend on the stage count
    other = vo.build_vit_stages(vo.VitSpec(), [2, 6], d_prime=1, n=3, seed=42)
    np.testing.assert_array_equal(stages[0].block[0]["wqkv"], other[0].block[0]["wqkv"])
    b0 = 1 / math.sqrt(384)
    assert np.abs(stages[1].block[0]["wqkv"]).max() <= b0


def test_local_step_follows_reference_update():
    st = vo.build_vit_stages(SPEC, [2, 1], d_prime=1, n=1, seed=3)[1]
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, SPEC.tokens, SPEC.dim))
    y = np.array([1, 4])
    before = [p.copy() for p in st.params()]
    _, _, _, grads = vo.local_grads(st, x, y)
    vo.local_step(st, x, y, 0.05, 0.001, 10, 0.9, 1e-4)
    lr = cosine_lr(0, 0.05, 0.001, 10)
    for p0, p1, g in zip(before, st.params(), grads):
        th, v = p0.copy(), np.zeros_like(p0)
        nesterov_update(th, v, g, lr, 0.9, 1e-4)
        np.testing.assert_allclose(p1, th, rtol=0, atol=1e-14)
    assert st.step_count == 1
