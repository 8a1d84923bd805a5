"""Pin the ResNet oracle's manual backward against torch.autograd (float64)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import resnet_oracle as ro
from ppll_oracle import cosine_lr, nesterov_update

SPEC = ro.ResNetSpec(n=1, image=8, channels=3, widths=(4, 8, 16), classes=5)


def _torch_loss(st, x_in, y):
    P = [torch.tensor(a, dtype=torch.float64, requires_grad=True) for a in st.params()]
    it = iter(P)
    x = torch.tensor(x_in, dtype=torch.float64).permute(0, 3, 1, 2)     # NCHW for torch

    def conv(x, wflat, k, stride, cin, cout):
        w = wflat.reshape(k, k, cin, cout).permute(3, 2, 0, 1)          # (r,s,c,o) -> (o,c,r,s)
        return F.conv2d(x, w, stride=stride, padding=(k - 1) // 2)

    def bn(z, g, b):
        return F.batch_norm(z, None, None, g, b, training=True, eps=ro.BN_EPS)

    if st.stem is not None:
        w, g, b = next(it), next(it), next(it)
        x = torch.relu(bn(conv(x, w, 3, 1, SPEC.channels, SPEC.widths[0]), g, b))
    for (cin, cout, stride, _), p in st.blocks:
        w1, g1, b1, w2, g2, b2 = [next(it) for _ in range(6)]
        h = torch.relu(bn(conv(x, w1, 3, stride, cin, cout), g1, b1))
        h = bn(conv(h, w2, 3, 1, cout, cout), g2, b2)
        if "ws" in p:
            ws, gs, bs = next(it), next(it), next(it)
            sc = bn(conv(x, ws, 1, stride, cin, cout), gs, bs)
        else:
            sc = x
        x = torch.relu(h + sc)
    C = x.shape[1]
    for _ in st.aux:
        w, g, b = next(it), next(it), next(it)
        x = torch.relu(bn(conv(x, w, 3, 1, C, C), g, b))
    hw, hb = next(it), next(it)
    logits = x.mean(dim=(2, 3)) @ hw + hb
    return F.cross_entropy(logits, torch.tensor(y)), P


@pytest.mark.parametrize("j", [0, 1, 2])
def test_manual_backward_matches_autograd(j):
    stages = ro.build_resnet_stages(SPEC, 3, d_prime=1, n_int=2, seed=7)
    st = stages[j]
    rng = np.random.default_rng(j)
    if j == 0:
        x = rng.standard_normal((3, 8, 8, 3))
    else:
        c, h = ro.stage_out_geometry(SPEC, stages[j - 1].blocks and
                                     [b for b in range(SPEC.n_blocks)][:sum(len(s.blocks) for s in stages[:j])])
        x = rng.standard_normal((3, h, h, c))
    y = rng.integers(0, SPEC.classes, 3)
    loss, x_out, logits, grads = ro.local_grads(st, x, y)
    tl, P = _torch_loss(st, x, y)
    tl.backward()
    assert abs(loss - tl.item()) < 1e-12
    names = st.param_list()
    assert len(grads) == len(P) == len(names)
    for (grp, key, _), g, p in zip(names, grads, P):
        np.testing.assert_allclose(g, p.grad.numpy(), rtol=1e-8, atol=1e-10, err_msg=f"{grp}.{key}")


def test_split_and_geometry():
    s32 = ro.ResNetSpec(n=5)
    split = ro.resnet_split(s32, 4)
    assert [len(b) for b in split] == [3, 4, 4, 4]
    # boundary activations of the FLOP-balanced ResNet-32 split
    assert [ro.stage_out_geometry(s32, b) for b in split[:3]] == [(16, 32), (32, 16), (64, 8)]
    s110 = ro.ResNetSpec(n=18)
    assert [len(b) for b in ro.resnet_split(s110, 8)] == [6, 7, 7, 7, 7, 7, 7, 6]   # 55 units
    assert ro.block_geometry(s32, 5) == (16, 32, 2, 32)
    assert ro.block_geometry(s32, 6) == (32, 32, 1, 16)


def test_local_step_update():
    st = ro.build_resnet_stages(SPEC, 2, d_prime=1, n_int=1, seed=3)[1]
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 8, 8, 4))      # output of [stem, block0]: 4 ch at 8x8
    y = np.array([1, 4])
    before = [p.copy() for p in st.params()]
    _, _, _, grads = ro.local_grads(st, x, y)
    ro.local_step(st, x, y, 0.05, 0.001, 10, 0.9, 1e-4)
    lr = cosine_lr(0, 0.05, 0.001, 10)
    for p0, p1, g in zip(before, st.params(), grads):
        th, v = p0.copy(), np.zeros_like(p0)
        nesterov_update(th, v, g, lr, 0.9, 1e-4)
        np.testing.assert_allclose(p1, th, rtol=0, atol=1e-14)
