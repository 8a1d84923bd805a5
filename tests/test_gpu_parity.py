"""GPU parity tests: the CUDA path (through the C-ABI) against the oracle and
the reference's golden vectors.

Tolerances (stated):
  * integer bookkeeping (batch ids, FIFO order, counts, staleness bounds,
    deterministic trace): bit-exact;
  * fp32 parity mode vs the fp64 reference: per-step loss |Δ| <= 5e-6 (x
    max(1,|loss|)); final weights max|ΔW| / max|W| <= 5e-3;
  * bf16 tensor-core mode: per-step loss |Δ| <= 2e-2 relative; weights
    max|ΔW| / max|W| <= 5e-2;
  * device pipeline vs device round-robin vs device sequential: bitwise.
"""
import json
import os

import numpy as np
import pytest
import torch

import paper_2411_12780_b200 as lp
import ppll_oracle as orc
from conftest import GOLDEN
from paper_2411_12780_b200 import _native as N

pytestmark = pytest.mark.gpu

CASES = ["mlp_s1", "mlp_s2", "mlp_s4", "mlp_s3_wide_aux", "mlp_s4_odd"]
TOL = {"fp32": (5e-6, 5e-3), "bf16": (2e-2, 5e-2)}


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    yield


def _mods(z, precision, total_steps=None):
    dims = tuple(int(d) for d in z["dims"])
    spec = lp.NetworkSpec(dims)
    plan = lp.partition(spec, int(z["s"]))
    ahw = int(z["aux_hidden_width"])
    hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001,
                           total_steps=total_steps or int(z["steps"]), momentum=0.9,
                           weight_decay=1e-4, seed=int(z["seed"]),
                           aux_hidden_width=None if ahw < 0 else ahw, precision=precision)
    return lp.build_modules(spec, plan, int(z["d_prime"]), int(z["interval"]), hyper)


def _flat(m):
    return np.concatenate([p.data.ravel() for p in m.parameters()])


# --- primitives through the C-ABI ------------------------------------------------

SHAPES = [(7, 5, 3), (64, 64, 64), (128, 3072, 1024), (100, 200, 10), (256, 384, 1152),
          (128, 1024, 1024), (33, 17, 29)]


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("M,K,Nn", SHAPES)
def test_linear_ops_match_torch_fp32(dtype, M, K, Nn):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + K)
    tdt = torch.float32 if dtype == "fp32" else torch.bfloat16
    code = N.F32 if dtype == "fp32" else N.BF16
    X = torch.randn(M, K, device="cuda", generator=g).to(tdt)
    W = (torch.randn(K, Nn, device="cuda", generator=g) / K ** 0.5).to(tdt)
    b = torch.randn(Nn, device="cuda", generator=g)
    dY = torch.randn(M, Nn, device="cuda", generator=g).to(tdt)
    Xm = torch.relu(X.float()).to(tdt)   # mask source with exact zeros
    lib = N.load()
    s = torch.cuda.current_stream().cuda_stream
    Y = torch.empty(M, Nn, device="cuda", dtype=tdt)
    Y2 = torch.empty_like(Y)
    N.check(lib.ppll_linear_fwd(M, K, Nn, X.data_ptr(), K, W.data_ptr(), b.data_ptr(),
                                Y.data_ptr(), Nn, Y2.data_ptr(), Nn, 1, code, s), "fwd")
    dX = torch.empty(M, K, device="cuda", dtype=tdt)
    N.check(lib.ppll_linear_dgrad(M, K, Nn, dY.data_ptr(), Nn, W.data_ptr(), Xm.data_ptr(), K,
                                  dX.data_ptr(), K, code, s), "dgrad")
    dW = torch.empty(K, Nn, device="cuda")
    db = torch.empty(Nn, device="cuda")
    N.check(lib.ppll_linear_wgrad(M, K, Nn, Xm.data_ptr(), K, dY.data_ptr(), Nn, dW.data_ptr(),
                                  db.data_ptr(), code, s), "wgrad")
    torch.cuda.synchronize()
    Xf, Wf, dYf, Xmf = X.double(), W.double(), dY.double(), Xm.double()
    refY = torch.relu(Xf @ Wf + b.double())
    refdX = (dYf @ Wf.T) * (Xmf > 0)
    refdW = Xmf.T @ dYf
    refdb = dYf.sum(0)
    rtol = 1e-5 if dtype == "fp32" else 2e-2

    def close(a, r):
        scale = r.abs().max().item() + 1e-12
        return (a.double() - r).abs().max().item() / scale

    assert close(Y, refY) < rtol
    assert torch.equal(Y, Y2)                       # dual store (fused push) is identical
    assert close(dX, refdX) < rtol
    assert bool(((Xmf > 0) | (dX.double() == 0)).all())   # mask: exact zeros
    assert close(dW, refdW) < rtol
    assert close(db, refdb) < 1e-5


def test_softmax_xent_kats_and_label_flag():
    z = lp.Tensor(np.zeros((3, 4)))
    assert lp.softmax_xent(z, np.array([0, 1, 3])).item() == pytest.approx(np.log(4), abs=1e-6)
    big = lp.Tensor(np.array([[1e4, 0.0], [0.0, 1e4]]))
    assert lp.softmax_xent(big, np.array([0, 1])).item() == pytest.approx(0.0, abs=1e-6)
    with pytest.raises(lp.LabelOutOfRange):
        lp.softmax_xent(z, np.array([0, 1, 4]))
    # the device flag path (range check left to the kernel)
    lib = N.load()
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    loss = torch.zeros(1, device="cuda")
    dz = torch.empty(3, 4, device="cuda")
    y = torch.tensor([0, 9, 1], device="cuda")
    N.check(lib.ppll_softmax_xent(3, 4, z.dev.data_ptr(), 4, y.data_ptr(), dz.data_ptr(), 4,
                                  loss.data_ptr(), None, err.data_ptr(), N.F32,
                                  torch.cuda.current_stream().cuda_stream), "xent")
    assert int(err.item()) & N.ERRBIT_LABEL


def test_softmax_xent_matches_oracle_random():
    rng = np.random.default_rng(3)
    for B, C in [(1, 2), (5, 10), (128, 10), (64, 100), (300, 7)]:
        zh = rng.standard_normal((B, C)) * 3
        yh = rng.integers(0, C, B)
        ref, gref = orc.softmax_xent(zh, yh)
        z = torch.tensor(zh, dtype=torch.float32, device="cuda")
        dz = torch.empty_like(z)
        loss = torch.zeros(1, device="cuda")
        N.check(N.load().ppll_softmax_xent(B, C, z.data_ptr(), C,
                                           torch.tensor(yh, device="cuda").data_ptr(),
                                           dz.data_ptr(), C, loss.data_ptr(), None, None, N.F32,
                                           torch.cuda.current_stream().cuda_stream), "xent")
        assert abs(loss.item() - ref) < 1e-5
        np.testing.assert_allclose(dz.cpu().numpy(), gref, atol=1e-7)


def test_nesterov_kats_and_recurrence():
    # test_optim.py:15-56 frozen values
    for th0, g, lr, mu, wd, want in [(1.0, 0.5, 0.1, 0.0, 0.0, 0.95), (0.0, 1.0, 1.0, 0.9, 0.0, -1.9),
                                     (10.0, 0.0, 1.0, 0.0, 1e-4, 9.999)]:
        p = lp.Tensor(np.array([th0]), track_grad=True)
        st = lp.OptimizerState([p], mu=mu, weight_decay=wd)
        p.grad = lp.Tensor(np.array([g]))
        lp.sgd_nesterov_step([p], st, lr)
        assert p.data[0] == pytest.approx(want, rel=1e-6)
        assert p.grad is None and st.step_count == 1
    p = lp.Tensor(np.array([0.0]), track_grad=True)
    st = lp.OptimizerState([p], mu=0.9, weight_decay=0.0)
    for _ in range(2):
        p.grad = lp.Tensor(np.array([1.0]))
        lp.sgd_nesterov_step([p], st, 1.0)
    assert p.data[0] == pytest.approx(-4.61, rel=1e-6)
    # all-or-nothing
    a, b = lp.Tensor(np.array([1.0]), track_grad=True), lp.Tensor(np.array([2.0]), track_grad=True)
    st = lp.OptimizerState([a, b])
    a.grad = lp.Tensor(np.array([1.0]))
    with pytest.raises(lp.MissingGradient):
        lp.sgd_nesterov_step([a, b], st, 0.1)
    assert a.data[0] == 1.0 and a.grad is not None and st.step_count == 0
    # random trajectories vs the oracle recurrence (optim.py:81-88)
    rng = np.random.default_rng(11)
    for _ in range(10):
        th0 = rng.normal(size=(37,))
        mu, wd, lr = rng.uniform(0, 0.95), rng.uniform(0, 0.01), rng.uniform(0.01, 0.2)
        p = lp.Tensor(th0.copy(), track_grad=True)
        st = lp.OptimizerState([p], mu=mu, weight_decay=wd)
        rt, rv = th0.copy(), np.zeros_like(th0)
        for _ in range(4):
            g = rng.normal(size=th0.shape)
            p.grad = lp.Tensor(g)
            lp.sgd_nesterov_step([p], st, lr)
            orc.nesterov_update(rt, rv, g, lr, mu, wd)
        np.testing.assert_allclose(p.data, rt, atol=1e-5)


# --- the local step vs the reference's golden vectors ---------------------------

@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("name", CASES)
def test_local_steps_match_reference_golden(name, precision):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    mods = _mods(z, precision)
    s, steps = int(z["s"]), int(z["steps"])
    for j, m in enumerate(mods):    # initial parameters: fp32 rounding of the fp64 draws
        np.testing.assert_allclose(_flat(m), z[f"init_{j}"], rtol=0, atol=1e-7)
    ltol, wtol = TOL[precision]
    losses = np.zeros((s, steps))
    for t in range(steps):
        h = lp.Tensor(z["xs"][t])
        for j, m in enumerate(mods):
            loss, h = lp.local_loss_and_update(m, h, z["ys"][t])
            losses[j, t] = loss
            if t == 0:
                ref = z[f"xout0_{j}"]
                err = np.abs(h.data - ref).max() / max(np.abs(ref).max(), 1e-6)
                assert err < (1e-5 if precision == "fp32" else 3e-2), (j, err)
    ref = z["losses"]
    if precision == "fp32":
        assert np.abs(losses - ref).max() <= ltol * max(1.0, np.abs(ref).max())
    else:
        assert (np.abs(losses - ref) / np.abs(ref)).max() <= ltol
    for j, m in enumerate(mods):
        fin, want = _flat(m), z[f"final_{j}"]
        assert np.abs(fin - want).max() / np.abs(want).max() <= wtol
        assert m.optimizer.step_count == int(z[f"step_count_{j}"])
        assert m.device_step() == steps


def test_full_m_config_fp32_losses():
    """(3072,1024,1024,1024,1024,10), s=4, B=128 vs the reference (3 steps)."""
    z = np.load(os.path.join(GOLDEN, "full_m.npz"))
    dims = (3072, 1024, 1024, 1024, 1024, 10)
    spec = lp.NetworkSpec(dims)
    mods = lp.build_modules(spec, lp.partition(spec, 4), 2, 3,
                            lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=100, seed=42))
    rng = np.random.default_rng(0)
    xs = rng.standard_normal((3, 128, 3072))
    ys = rng.integers(0, 10, size=(3, 128))
    losses = np.zeros((4, 3))
    for t in range(3):
        h = lp.Tensor(xs[t])
        for j, m in enumerate(mods):
            losses[j, t], h = lp.local_loss_and_update(m, h, ys[t])
    assert np.abs(losses - z["losses"]).max() <= 5e-6 * 3
    for j, m in enumerate(mods):
        f = _flat(m)
        np.testing.assert_allclose(f[:256], z[f"head_{j}"], atol=5e-5)


# --- local-step semantics (test_blocks.py:198-238) -------------------------------

def test_gradient_isolation_and_pre_step_output():
    z = np.load(os.path.join(GOLDEN, "mlp_s4.npz"))
    mods = _mods(z, "fp32", total_steps=10)
    before = [_flat(m) for m in mods]
    x = lp.Tensor(np.random.default_rng(8).normal(size=(5, mods[1].input_width)))
    expected = lp.block_forward(mods[1], x).data
    seen = []
    loss, x_out = lp.local_loss_and_update(mods[1], x, np.array([0, 1, 2, 3, 4]),
                                           on_output=seen.append)
    assert np.isfinite(loss)
    assert np.array_equal(x_out.data, expected)          # pre-update parameters
    assert len(seen) == 1 and seen[0] is x_out and not x_out.track_grad
    after = [_flat(m) for m in mods]
    for j in range(4):
        assert np.array_equal(before[j], after[j]) == (j != 1)
    with pytest.raises(ValueError):
        lp.local_loss_and_update(mods[0], lp.Tensor(np.zeros((2, 96)), track_grad=True),
                                 np.array([0, 1]))
    with pytest.raises(lp.DimensionMismatch):
        lp.block_forward(mods[0], lp.Tensor(np.zeros((2, 5))))


def test_label_error_and_step_out_of_range():
    z = np.load(os.path.join(GOLDEN, "mlp_s2.npz"))
    mods = _mods(z, "fp32", total_steps=1)
    before = _flat(mods[0])
    with pytest.raises(lp.LabelOutOfRange):
        lp.local_loss_and_update(mods[0], lp.Tensor(np.zeros((3, 48))), np.array([0, 99, 1]))
    assert np.array_equal(_flat(mods[0]), before) and mods[0].optimizer.step_count == 0
    x = lp.Tensor(np.ones((3, 48)))
    lp.local_loss_and_update(mods[0], x, np.array([0, 1, 2]))
    lp.local_loss_and_update(mods[0], x, np.array([0, 1, 2]))   # step 1 == total_steps: allowed
    with pytest.raises(lp.StepOutOfRange):
        lp.local_loss_and_update(mods[0], x, np.array([0, 1, 2]))


# --- the pipeline (runtime.py) -----------------------------------------------------

def _toy(n, width, classes, batch, seed):
    rng = np.random.default_rng(seed)
    return [(rng.normal(size=(batch, width)), rng.integers(0, classes, size=batch))
            for _ in range(n)]


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_device_pipeline_equals_roundrobin_equals_sequential(precision):
    z = np.load(os.path.join(GOLDEN, "mlp_s4.npz"))
    data = _toy(9, 96, 10, 16, 5)
    a, b, c = (_mods(z, precision, total_steps=20) for _ in range(3))
    ma = lp.run_epoch(lp.RunMode.PPLL, a, iter(data), lp.RunConfig(buffer_capacity=2))
    mb = lp.run_deterministic(lp.RunMode.PPLL, b, iter(data), lp.RunConfig(buffer_capacity=3))
    seq = [[] for _ in range(4)]
    for x, y in data:
        h = lp.Tensor(x)
        for j, m in enumerate(c):
            loss, h = lp.local_loss_and_update(m, h, y)
            seq[j].append(loss)
    assert ma.loss_history == mb.loss_history == seq
    for x, y, w in zip(a, b, c):
        assert np.array_equal(_flat(x), _flat(y)) and np.array_equal(_flat(x), _flat(w))
    assert ma.batches_processed == mb.batches_processed == [9] * 4
    assert sum(ma.staleness.values()) == 36 and all(0 <= k <= 2 for k in ma.staleness)
    assert all(1 <= hw <= 2 for hw in ma.buffer_high_water)
    assert ma.wall_time > 0 and all(0 < bt <= ma.wall_time for bt in ma.busy_time)


def test_pipeline_matches_reference_threaded_golden():
    """The reference's threaded run_epoch (golden) == our device pipeline."""
    z = np.load(os.path.join(GOLDEN, "threaded_ppll.npz"))
    dims = (24, 20, 16, 12, 6)
    spec = lp.NetworkSpec(dims)
    mods = lp.build_modules(spec, lp.partition(spec, 3), 2, 1,
                            lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=20, seed=3))
    data = list(zip(z["xs"], z["ys"]))
    m = lp.run_epoch(lp.RunMode.PPLL, mods, iter(data), lp.RunConfig(buffer_capacity=2))
    assert np.abs(np.array(m.loss_history) - z["losses"]).max() < 5e-6 * 3
    for j, mod in enumerate(mods):
        want = z[f"final_{j}"]
        assert np.abs(_flat(mod) - want).max() / np.abs(want).max() < 5e-3


def test_deterministic_traces_bit_exact():
    with open(os.path.join(GOLDEN, "roundrobin_traces.json")) as f:
        traces = json.load(f)
    for t in traces:
        s, n, M = t["s"], t["n"], t["M"]
        dims = (4,) + (5,) * s + (2,)
        spec = lp.NetworkSpec(dims)
        mods = lp.build_modules(spec, lp.partition(spec, s), 1, 1,
                                lp.Hyperparams(total_steps=64, seed=0))
        rng = np.random.default_rng(s * 100 + n)
        data = [(rng.standard_normal((3, 4)), rng.integers(0, 2, 3)) for _ in range(n)]
        m = lp.run_deterministic(lp.RunMode.PPLL, mods, iter(data), lp.RunConfig(buffer_capacity=M))
        assert m.wall_time == t["wall_time"]
        assert m.busy_time == t["busy_time"]
        assert m.batches_processed == t["batches_processed"]
        assert {str(k): v for k, v in sorted(m.staleness.items())} == t["staleness"]
        assert m.buffer_high_water == t["high_water"]
        assert m.n_batches == t["n_batches"]


def test_conservation_and_bounds_random_pipelines():
    rng = np.random.default_rng(0)
    for _ in range(6):
        s = int(rng.integers(2, 6))
        cap = int(rng.integers(1, 4))
        n = int(rng.integers(1, 12))
        dims = (4,) + tuple(int(rng.integers(3, 9)) for _ in range(s)) + (3,)
        spec = lp.NetworkSpec(dims)
        mods = lp.build_modules(spec, lp.partition(spec, s), 1, 1,
                                lp.Hyperparams(total_steps=64, seed=int(rng.integers(1000))))
        m = lp.run_epoch(lp.RunMode.PPLL, mods, iter(_toy(n, 4, 3, 6, int(rng.integers(99)))),
                         lp.RunConfig(buffer_capacity=cap))
        assert m.n_batches == n and m.batches_processed == [n] * s
        assert [len(h) for h in m.loss_history] == [n] * s
        assert sum(m.staleness.values()) == s * n
        assert all(0 <= k <= cap for k in m.staleness)
        assert all(1 <= hw <= cap for hw in m.buffer_high_water)


def test_worker_failure_surfaces_as_panic():
    spec = lp.NetworkSpec((4, 5, 4, 2))
    mods = lp.build_modules(spec, lp.partition(spec, 2), 1, 1, lp.Hyperparams(total_steps=8))
    with pytest.raises(lp.WorkerPanic) as err:
        lp.run_epoch(lp.RunMode.PPLL, mods, iter([(np.zeros((3, 4)), np.array([0, 9, 1]))]))
    assert err.value.stage_index in (0, 1)


def test_native_kernels_were_launched():
    before = N.launch_count()
    spec = lp.NetworkSpec((32, 16, 8))
    mods = lp.build_modules(spec, lp.partition(spec, 1), 0, 1, lp.Hyperparams(total_steps=4))
    lp.local_loss_and_update(mods[0], lp.Tensor(np.ones((4, 32))), np.array([0, 1, 2, 3]))
    assert N.launch_count() > before


# --- the tcgen05 engine specifically ---------------------------------------------

TC_SHAPES = [(128, 64, 64), (128, 3072, 1024), (256, 384, 1152), (100, 200, 96),
             (8320, 384, 1536), (130, 1024, 264), (1024, 1024, 1024),
             # long reductions: the weight gradient takes the cluster split-K path
             (8320, 1536, 384), (3000, 136, 72), (4736, 768, 3072)]


@pytest.mark.parametrize("M,K,Nn", TC_SHAPES)
def test_tcgen05_engine_matches_torch(M, K, Nn):
    lib = N.load()
    lib.ppll_set_gemm_engine(N.GEMM_TCGEN05)
    try:
        test_linear_ops_match_torch_fp32("bf16", M, K, Nn)
    finally:
        lib.ppll_set_gemm_engine(N.GEMM_AUTO)


@pytest.mark.parametrize("M,K,Nn", [(8320, 384, 1536), (3000, 136, 72), (131072, 144, 16)])
def test_wgrad_split_reduction_is_deterministic(M, K, Nn):
    """Split-K weight gradients (cluster DSMEM or workspace reduction) sum the
    K slices in a fixed order: two runs are bitwise identical."""
    g = torch.Generator(device="cuda").manual_seed(M + K + Nn)
    X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    dY = torch.randn(M, Nn, device="cuda", generator=g).bfloat16()
    lib = N.load()
    s = torch.cuda.current_stream().cuda_stream
    outs = []
    for _ in range(2):
        dW = torch.full((K, Nn), float("nan"), device="cuda")
        N.check(lib.ppll_linear_wgrad(M, K, Nn, X.data_ptr(), K, dY.data_ptr(), Nn,
                                      dW.data_ptr(), None, N.BF16, s), "wgrad")
        outs.append(dW)
    torch.cuda.synchronize()
    ref = X.double().T @ dY.double()
    assert torch.equal(outs[0], outs[1])
    assert (outs[0].double() - ref).abs().max().item() / ref.abs().max().item() < 1e-2


@pytest.mark.parametrize("engine", ["tcgen05", "simt"])
@pytest.mark.parametrize("M,K,Nn", [(1040, 384, 1536), (200, 96, 136)])
def test_gelu_epilogues_match_torch(engine, M, K, Nn):
    """Transformer-layer epilogues: residual, GELU(erf), pre-activation /
    GELU-derivative stores, GELU-gradient and stored-derivative masks."""
    g = torch.Generator(device="cuda").manual_seed(M + Nn)
    X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(K, Nn, device="cuda", generator=g) / K ** 0.5).bfloat16()
    b = torch.randn(Nn, device="cuda", generator=g)
    R = torch.randn(M, Nn, device="cuda", generator=g).bfloat16()
    dY = torch.randn(M, Nn, device="cuda", generator=g).bfloat16()
    Mk = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    lib = N.load()
    lib.ppll_set_gemm_engine(N.GEMM_TCGEN05 if engine == "tcgen05" else N.GEMM_SIMT)
    s = torch.cuda.current_stream().cuda_stream
    try:
        outs = {}
        for act in (2, 3):
            Y = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
            P = torch.empty_like(Y)
            N.check(lib.ppll_linear_fwd_ex(M, K, Nn, X.data_ptr(), K, W.data_ptr(), b.data_ptr(),
                                           R.data_ptr(), Nn, act, P.data_ptr(), Nn, Y.data_ptr(),
                                           Nn, None, 0, N.BF16, s), "fwd_ex")
            outs[act] = (Y, P)
        dX = {}
        for mode in (2, 3):
            d = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
            N.check(lib.ppll_linear_dgrad_ex(M, K, Nn, dY.data_ptr(), Nn, W.data_ptr(),
                                             Mk.data_ptr(), K, mode, d.data_ptr(), K, N.BF16, s),
                    "dgrad_ex")
            dX[mode] = d
        torch.cuda.synchronize()
    finally:
        lib.ppll_set_gemm_engine(N.GEMM_AUTO)
    u = X.double() @ W.double() + b.double() + R.double()
    gelu = torch.nn.functional.gelu(u)
    cdf = 0.5 * (1 + torch.erf(u / 2 ** 0.5))
    dgelu = cdf + u * torch.exp(-0.5 * u * u) / (2 * torch.pi) ** 0.5

    def rel(a, r):
        return (a.double() - r).abs().max().item() / (r.abs().max().item() + 1e-12)

    assert rel(outs[2][0], gelu) < 1e-2 and rel(outs[2][1], u) < 1e-2
    assert rel(outs[3][0], gelu) < 1e-2 and rel(outs[3][1], dgelu) < 1e-2
    mk = Mk.double()
    dmk = 0.5 * (1 + torch.erf(mk / 2 ** 0.5)) + mk * torch.exp(-0.5 * mk * mk) / (2 * torch.pi) ** 0.5
    base = dY.double() @ W.double().T
    assert rel(dX[2], base * dmk) < 1e-2
    assert rel(dX[3], base * mk) < 1e-2


# --- the paper's baselines: E2E and naive PP (runtime.py:248-284, 359-382) -------

@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("tag", ["s2", "s4", "s3"])
def test_e2e_and_naive_pp_match_reference(tag, precision):
    """run_epoch / run_deterministic in E2E and NAIVE_PP modes on the device
    against the reference's (bitwise-identical) four runs; the four device
    runs are bitwise identical to each other; aux heads are never touched."""
    z = np.load(os.path.join(GOLDEN, "e2e_naive.npz"))
    dims = tuple(int(d) for d in z[f"{tag}_dims"])
    s = int(z[f"{tag}_s"])
    data = list(zip(z[f"{tag}_xs"], z[f"{tag}_ys"]))
    spec = lp.NetworkSpec(dims)
    ltol, wtol = TOL[precision]
    runs = []
    for mode in (lp.RunMode.E2E, lp.RunMode.NAIVE_PP):
        for runner in (lp.run_deterministic, lp.run_epoch):
            hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=10, seed=42,
                                   precision=precision)
            mods = lp.build_modules(spec, lp.partition(spec, s), 2, 3, hyper)
            init = [_flat(m) for m in mods]
            met = runner(mode, mods, iter(data), lp.RunConfig(buffer_capacity=2))
            runs.append((met, mods, init))
    ref_l = z[f"{tag}_losses"]
    for met, mods, init in runs:
        assert met.n_batches == len(data) and met.batches_processed == [len(data)] * s
        assert [len(h) for h in met.loss_history] == list(z[f"{tag}_n_losses"])
        got = np.array(met.loss_history[-1])
        if precision == "fp32":
            assert np.abs(got - ref_l).max() <= ltol * max(1.0, np.abs(ref_l).max())
        else:
            assert (np.abs(got - ref_l) / np.abs(ref_l)).max() <= ltol
        for j, m in enumerate(mods):
            fin, want = _flat(m), z[f"{tag}_final_{j}"]
            assert np.abs(fin - want).max() / np.abs(want).max() <= wtol
            nb = sum(p.data.size for p in m.block_parameters())
            assert np.array_equal(fin[nb:], init[j][nb:])          # aux untouched
            assert m.optimizer.step_count == int(z[f"{tag}_step_{j}"]) == m.device_step()
    base = runs[0]
    for met, mods, _ in runs[1:]:
        assert met.loss_history == base[0].loss_history
        for a, b in zip(mods, base[1]):
            assert np.array_equal(_flat(a), _flat(b))


# --- data path and evaluation ---------------------------

def _mlp_dataset(n=300, dims=(96, 64, 64, 48, 40, 10), seed=3):
    rng = np.random.default_rng(seed)
    return lp.Dataset(rng.standard_normal((n, dims[0])), rng.integers(0, dims[-1], n),
                      dims[-1])


def test_device_dataset_batches_equal_host_batches():
    ds = _mlp_dataset()
    dd = lp.DeviceDataset(ds)
    for shuffle, seed in ((True, 4), (False, 0)):
        host = list(lp.batches(ds, 64, shuffle=shuffle, seed=seed))
        dev = list(dd.batches(64, shuffle=shuffle, seed=seed))
        assert len(host) == len(dev) == 5
        for (hx, hy), (dx, dy) in zip(host, dev):
            assert np.array_equal(dx.cpu().numpy(), hx.astype(np.float32))
            assert np.array_equal(dy.cpu().numpy(), hy)
    bx, _ = next(dd.batches(64, True, 4, dtype=torch.bfloat16))
    hx, _ = next(iter(lp.batches(ds, 64, True, 4)))
    assert torch.equal(bx, torch.as_tensor(hx, dtype=torch.float32).bfloat16().cuda())


def test_device_idx_dataset_u8_gather(tmp_path):
    """An IDX dataset lives in HBM as its pixel bytes; the per-batch /255
    (ppll_gather_rows_u8) reproduces load_idx's features exactly in fp32
    and as their bf16 rounding."""
    import struct
    rng = np.random.default_rng(3)
    count, rows, cols = 203, 32, 48          # 1536 features: the 16-B vector path
    for c in (cols, 7):                       # and a ragged width (scalar path)
        pix = rng.integers(0, 256, (count, rows * c), dtype=np.uint8)
        lab = rng.integers(0, 10, count, dtype=np.uint8)
        (tmp_path / "i").write_bytes(struct.pack(">IIII", 0x803, count, rows, c) + pix.tobytes())
        (tmp_path / "l").write_bytes(struct.pack(">II", 0x801, count) + lab.tobytes())
        ds = lp.load_idx(tmp_path / "i", tmp_path / "l")
        dd = lp.DeviceDataset(ds)
        assert dd.features.dtype == torch.uint8
        host = list(lp.batches(ds, 64, shuffle=True, seed=5))
        dev = list(dd.batches(64, shuffle=True, seed=5))
        dev16 = list(dd.batches(64, shuffle=True, seed=5, dtype=torch.bfloat16))
        assert len(host) == len(dev) == 4
        for (hx, hy), (dx, dy), (bx, _) in zip(host, dev, dev16):
            assert np.array_equal(dx.cpu().numpy(), hx.astype(np.float32))
            assert np.array_equal(dy.cpu().numpy(), hy)
            assert torch.equal(bx, dx.bfloat16())


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_run_epoch_device_batches_equal_host_batches(precision):
    ds = _mlp_dataset()
    spec = lp.NetworkSpec((96, 64, 64, 48, 40, 10))
    outs = []
    for src in ("host", "device", "pinned"):
        hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=20, seed=42,
                               precision=precision)
        mods = lp.build_modules(spec, lp.partition(spec, 4), 2, 3, hyper)
        if src == "host":
            it = lp.batches(ds, 64, True, 7)
        elif src == "device":
            it = lp.DeviceDataset(ds).batches(64, True, 7)
        else:   # caller-pinned host tensors: copied straight to the device
            it = [(torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).pin_memory(),
                   torch.from_numpy(np.asarray(y, dtype=np.int64)).pin_memory())
                  for x, y in lp.batches(ds, 64, True, 7)]
        met = lp.run_epoch(lp.RunMode.PPLL, mods, it)
        outs.append((met.loss_history, [_flat(m) for m in mods]))
    for o in outs[1:]:
        assert outs[0][0] == o[0]
        for a, b in zip(outs[0][1], o[1]):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_evaluate_matches_oracle_forward(precision):
    """evaluate (harness.py:121-131) on the device == argmax of an fp64
    forward of the same (device) parameters, row for row up to ties."""
    dims = (96, 64, 64, 48, 40, 10)
    ds = _mlp_dataset(n=700, dims=dims)
    spec = lp.NetworkSpec(dims)
    hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=20, seed=42, precision=precision)
    mods = lp.build_modules(spec, lp.partition(spec, 4), 2, 3, hyper)
    lp.run_epoch(lp.RunMode.PPLL, mods, lp.batches(ds, 100, True, 1))
    acc = lp.evaluate(mods, ds, chunk=256)
    h = ds.features
    for m in mods:
        for layer in m.layers:
            h = h @ layer.W.data.astype(np.float64) + layer.b.data.astype(np.float64)
            if layer.relu_after:
                h = np.maximum(h, 0.0)
    ref = float((h.argmax(axis=1) == ds.labels).mean())
    tol = 0.0 if precision == "fp32" else 0.03
    assert abs(acc - ref) <= tol + 2.0 / ds.n, (acc, ref)
    mem = lp.device_memory(mods[0])
    assert mem["params_state_bytes"] > 0 and mem["workspace_bytes"] >= 0


def test_calibrate_feeds_the_schedule_simulator():
    """costs.calibrate measures every stage on the device; the simulated
    one-stage-per-GPU PPLL schedule is governed by the slowest stage."""
    spec = lp.NetworkSpec((96, 64, 64, 48, 40, 10))
    hyper = lp.Hyperparams(total_steps=10 ** 6, seed=1)
    mods = lp.build_modules(spec, lp.partition(spec, 4), 2, 3, hyper)
    prof = lp.calibrate(mods, 32, reps=5)
    assert len(prof) == 4 and all(p.cycle > 0 and p.f > 0 for p in prof)
    r = lp.simulate_schedule(prof, lp.CommModel(), "ppll", 32, 2)
    assert r.steady_batch_time == pytest.approx(max(p.cycle for p in prof), rel=1e-6)
    assert min(r.idle_fraction(4)) < 1e-6


def test_run_experiment_matches_reference(tmp_path):
    """harness.run_experiment on the device (all three modes, 2 epochs, blobs
    and spirals) against the reference's own run (tests/golden/experiment.json):
    losses within the fp32 tolerance, accuracies within 2 rows, the float-count
    memory proxy and the deterministic staleness exact."""
    import json
    cases = json.load(open(os.path.join(GOLDEN, "experiment.json")))
    for case in cases:
        kw = {k: tuple(v) if isinstance(v, list) else v for k, v in case["config"].items()}
        cfg = lp.ExperimentConfig(**kw)
        recs, rep = lp.run_experiment(cfg, deterministic=True)
        n = cfg.n_per_class * (cfg.classes if cfg.dataset == "blobs" else 2)
        assert len(recs) == len(case["records"])
        for r, g in zip(recs, case["records"]):
            assert (r.mode, r.epoch) == (g[0], g[1])
            assert abs(r.mean_loss - g[2]) <= 5e-5, (r, g)
            assert abs(r.train_acc - g[3]) <= 2.0 / n and abs(r.test_acc - g[4]) <= 2.0 / n, (r, g)
            assert (r.params_max_stage, r.activations_max_stage) == (g[5], g[6])
            assert abs(r.mean_staleness - g[7]) < 1e-12
        assert [s.mode for s in rep.summaries] == case["modes"] and rep.stages == case["stages"]
        assert rep.measured_k > 0 and rep.ppll_over_pp_throughput > 0
        lp.write_metrics_csv(recs, tmp_path / "metrics.csv")
        assert lp.report_table(rep).count("\n") == len(cfg.modes) + 2
    # the threaded device pipeline trains bit-identically to the deterministic replay
    cfg = lp.ExperimentConfig(**{k: tuple(v) if isinstance(v, list) else v
                                 for k, v in cases[0]["config"].items()})
    thr, _ = lp.run_experiment(cfg)
    det, _ = lp.run_experiment(cfg, deterministic=True)
    for a, b in zip(thr, det):
        assert (a.mean_loss, a.train_acc, a.test_acc) == (b.mean_loss, b.train_acc, b.test_acc)


def test_run_experiment_on_idx_matches_reference(tmp_path):
    """The IDX path end to end: load_idx -> HBM-resident pixel bytes -> the
    device u8 gather -> run_experiment (all modes), against the reference's
    own run on the same files (tests/golden/experiment_idx.json)."""
    import json
    g = json.load(open(os.path.join(GOLDEN, "experiment_idx.json")))
    (tmp_path / "i.idx").write_bytes(bytes(g["images"]))
    (tmp_path / "l.idx").write_bytes(bytes(g["labels"]))
    kw = {k: tuple(v) if isinstance(v, list) else v for k, v in g["config"].items()}
    cfg = lp.ExperimentConfig(idx_train_images=str(tmp_path / "i.idx"),
                              idx_train_labels=str(tmp_path / "l.idx"), **kw)
    recs, rep = lp.run_experiment(cfg, deterministic=True)
    n = len(g["labels"]) - 8
    assert len(recs) == len(g["records"])
    for r, ref in zip(recs, g["records"]):
        assert (r.mode, r.epoch) == (ref[0], ref[1])
        assert abs(r.mean_loss - ref[2]) <= 5e-5, (r, ref)
        assert abs(r.train_acc - ref[3]) <= 2.0 / n and abs(r.test_acc - ref[4]) <= 2.0 / n
        assert (r.params_max_stage, r.activations_max_stage) == (ref[5], ref[6])
        assert abs(r.mean_staleness - ref[7]) < 1e-12
