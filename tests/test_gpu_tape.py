"""The device GradTape (tensor.py:96-278 restated on the device; the C-ABI
ppll_ew / ppll_colsum / ppll_sum_all / ppll_linear_dgrad / _wgrad adjoints)
against the reference's tensor tests (pkg/tests/test_tensor.py): the same
KATs and lifecycle rules, fp32 device arithmetic (tolerances 1e-6 relative
where the reference asserts 1e-15 in float64)."""
import math
import threading

import numpy as np
import pytest
import torch

import paper_2411_12780_b200 as lp

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def close(a, b, rtol=1e-6):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return np.allclose(a, b, rtol=rtol, atol=rtol * max(1.0, np.abs(b).max()))


def test_forward_kats():
    assert np.array_equal(lp.matmul(lp.Tensor([[1.0, 2.0], [3.0, 4.0]]),
                                    lp.Tensor([[5.0, 6.0], [7.0, 8.0]])).data, [[19, 22], [43, 50]])
    assert np.array_equal(lp.relu(lp.Tensor([[-1.0, 0.0, 2.0]])).data, [[0.0, 0.0, 2.0]])
    m = lp.Tensor([[1.0, 2.0], [3.0, 4.0]])
    assert np.array_equal(lp.bias_add(m, lp.Tensor([10.0, 20.0])).data, [[11, 22], [13, 24]])
    x = lp.Tensor([[1.0, -2.0], [3.0, 0.5]])
    assert np.array_equal(lp.scale(x, -2.0).data, [[-2.0, 4.0], [-6.0, -1.0]])
    assert lp.sum_all(x).item() == 2.5
    with pytest.raises(lp.DimensionMismatch):
        lp.add(lp.Tensor(np.zeros((2, 3))), lp.Tensor(np.zeros(3)))
    with pytest.raises(lp.DimensionMismatch):
        lp.bias_add(m, lp.Tensor([1.0, 2.0, 3.0]))


def test_xent_kats_and_gradient():
    loss = lp.softmax_xent(lp.Tensor(np.zeros((3, 4))), np.array([0, 1, 3]))
    assert abs(loss.item() - math.log(4.0)) < 1e-6
    big = lp.softmax_xent(lp.Tensor([[1000.0, 0.0], [0.0, 1000.0]]), np.array([0, 1]))
    assert np.isfinite(big.item()) and big.item() < 1e-6
    rng = np.random.default_rng(11)
    z = rng.normal(size=(3, 5))
    logits = lp.Tensor(z, track_grad=True)
    y = np.array([4, 0, 2])
    with lp.GradTape():
        lp.backward(lp.softmax_xent(logits, y))
    p = np.exp(z - z.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    p[np.arange(3), y] -= 1.0
    assert close(logits.grad, p / 3, 1e-5)


def test_primitive_adjoints():
    x = lp.Tensor(np.arange(6.0).reshape(2, 3), track_grad=True)
    with lp.GradTape():
        lp.backward(lp.sum_all(x))
    assert np.array_equal(x.grad, np.ones((2, 3)))
    x = lp.Tensor([[-1.0, 0.0, 2.0]], track_grad=True)
    with lp.GradTape():
        lp.backward(lp.sum_all(lp.relu(x)))
    assert np.array_equal(x.grad, [[0.0, 0.0, 1.0]])          # 0 at the kink
    rng = np.random.default_rng(0)
    a = lp.Tensor(rng.normal(size=(3, 4)), track_grad=True)
    b = lp.Tensor(rng.normal(size=(4, 2)), track_grad=True)
    with lp.GradTape():
        lp.backward(lp.sum_all(lp.matmul(a, b)))
    ones = np.ones((3, 2))
    assert close(a.grad, ones @ b.data.T) and close(b.grad, a.data.T @ ones)
    m = lp.Tensor(np.zeros((5, 3)), track_grad=True)
    v = lp.Tensor(np.zeros(3), track_grad=True)
    with lp.GradTape():
        lp.backward(lp.sum_all(lp.bias_add(m, v)))
    assert np.array_equal(v.grad, [5.0, 5.0, 5.0]) and np.array_equal(m.grad, np.ones((5, 3)))
    x = lp.Tensor([[2.0, 3.0]], track_grad=True)
    with lp.GradTape():
        lp.backward(lp.sum_all(lp.add(x, x)))
    assert np.array_equal(x.grad, [[2.0, 2.0]])                # accumulation


def test_mlp_chain_matches_torch_autograd():
    """A two-layer MLP step through the tape equals torch.autograd (fp64)."""
    rng = np.random.default_rng(3)
    X, W1, b1, W2, b2 = (rng.normal(size=s) for s in ((16, 12), (12, 8), (8,), (8, 5), (5,)))
    y = rng.integers(0, 5, 16)
    P = [lp.Tensor(a, track_grad=True) for a in (W1, b1, W2, b2)]
    with lp.GradTape():
        h = lp.relu(lp.bias_add(lp.matmul(lp.Tensor(X), P[0]), P[1]))
        loss = lp.softmax_xent(lp.bias_add(lp.matmul(h, P[2]), P[3]), y)
        lp.backward(loss)
    T = [torch.tensor(a, requires_grad=True) for a in (W1, b1, W2, b2)]
    ref = torch.nn.functional.cross_entropy(
        torch.relu(torch.tensor(X) @ T[0] + T[1]) @ T[2] + T[3], torch.tensor(y))
    ref.backward()
    assert abs(loss.item() - ref.item()) < 1e-5
    for p, t in zip(P, T):
        assert close(p.grad, t.grad.numpy(), 1e-4)


def test_tape_lifecycle():
    x = lp.Tensor([[1.0, -2.0]], track_grad=True)
    with lp.GradTape() as tape:
        loss = lp.sum_all(lp.relu(x))
        lp.backward(loss)
    assert tape.consumed and not tape.nodes
    with pytest.raises(lp.EmptyTape):
        lp.backward(loss)
    with pytest.raises(lp.EmptyTape):
        lp.backward(lp.Tensor(np.asarray(1.0)))
    x = lp.Tensor(np.ones((2, 2)), track_grad=True)
    with lp.GradTape() as tape:
        h = x
        for _ in range(12):
            h = lp.scale(h, 1.01)
        loss = lp.sum_all(h)
        n = len(tape.nodes)
        with pytest.raises(lp.NotScalar):
            lp.backward(h)
        lp.backward(loss)
    assert n == 13 and tape.adjoints_run == 13
    # unreachable branch skipped; no recording without a tape; detach cuts
    x = lp.Tensor([[1.0, 2.0]], track_grad=True)
    y = lp.Tensor([[3.0, 4.0]], track_grad=True)
    with lp.GradTape() as tape:
        loss = lp.sum_all(lp.scale(x, 3.0))
        side = lp.relu(y)
        lp.backward(loss)
    assert y.grad is None and side.grad is None and tape.adjoints_run == 2
    assert np.array_equal(x.grad, [[3.0, 3.0]])
    out = lp.relu(lp.Tensor([[1.0, 2.0]], track_grad=True))
    assert not out.track_grad and out._tape is None
    x = lp.Tensor(np.ones((2, 2)), track_grad=True)
    with lp.GradTape():
        h = lp.scale(x, 2.0)
        d = h.detach()
        assert not d.track_grad and d._tape is None
        lp.backward(lp.sum_all(h))
    assert np.array_equal(x.grad, 2.0 * np.ones((2, 2)))


def test_backward_from_and_threads():
    rng = np.random.default_rng(5)
    x = lp.Tensor(rng.normal(size=(3, 2)), track_grad=True)
    w = lp.Tensor(rng.normal(size=(2, 4)), track_grad=True)
    with lp.GradTape():
        h = lp.matmul(x, w)
    g = rng.normal(size=(3, 4))
    lp.backward_from(h, g)
    assert close(w.grad, x.data.T @ g) and close(x.grad, g @ w.data.T)
    with lp.GradTape():
        h = lp.scale(lp.Tensor(np.ones((2, 2)), track_grad=True), 1.0)
    with pytest.raises(lp.DimensionMismatch):
        lp.backward_from(h, np.ones((3, 2)))
    barrier = threading.Barrier(2)
    grads = {}

    def work(tag, factor):
        torch.cuda.set_device(0)
        barrier.wait()
        t = lp.Tensor(np.ones((1, 3)), track_grad=True)
        with lp.GradTape():
            lp.backward(lp.sum_all(lp.scale(t, factor)))
        grads[tag] = t.grad.copy()

    ths = [threading.Thread(target=work, args=("a", 2.0)),
           threading.Thread(target=work, args=("b", -5.0))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert np.array_equal(grads["a"], 2.0 * np.ones((1, 3)))
    assert np.array_equal(grads["b"], -5.0 * np.ones((1, 3)))


def test_non_finite_guards():
    with pytest.raises(lp.NonFiniteError):
        lp.Tensor([np.nan])
    big = lp.Tensor([[1e30]])
    with pytest.raises(lp.NonFiniteError):
        lp.matmul(big, lp.Tensor([[1e10]]))
    with pytest.raises(lp.NonFiniteError):
        lp.scale(big, 1e10)


def test_tape_gradients_drive_sgd_nesterov_step():
    """GradTape gradients feed the reference optimizer entry point."""
    rng = np.random.default_rng(8)
    W = lp.Tensor(rng.normal(size=(6, 4)), track_grad=True)
    b = lp.Tensor(rng.normal(size=(4,)), track_grad=True)
    st = lp.OptimizerState([W, b], mu=0.9, weight_decay=1e-4)
    X = rng.normal(size=(10, 6))
    y = rng.integers(0, 4, 10)
    w0, b0 = W.data.copy(), b.data.copy()
    with lp.GradTape():
        lp.backward(lp.softmax_xent(lp.bias_add(lp.matmul(lp.Tensor(X), W), b), y))
    gW, gb = W.grad.data.copy(), b.grad.data.copy()
    lp.sgd_nesterov_step([W, b], st, 0.1)
    for p, p0, g in ((W, w0, gW), (b, b0, gb)):
        gp = g + 1e-4 * p0
        v = gp
        assert close(p.data, p0 - 0.1 * (gp + 0.9 * v), 1e-5)
        assert p.grad is None
