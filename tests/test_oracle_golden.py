"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/gen_golden.py imports /root/reference's locopipe) and against
the reference tests' own known-answer values.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import ppll_oracle as orc
from conftest import GOLDEN

CASES = ["mlp_s1", "mlp_s2", "mlp_s4", "mlp_s3_wide_aux", "mlp_s4_odd"]
HYPER = dict(lr0=0.05, lr_min=0.001, mu=0.9, wd=1e-4)


def _load(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def _stages_for(z):
    dims = tuple(int(d) for d in z["dims"])
    s = int(z["s"])
    bnd = orc.partition(dims, s)
    ahw = int(z["aux_hidden_width"])
    st = orc.build_stages(dims, bnd, int(z["d_prime"]), int(z["interval"]),
                          int(z["seed"]), None if ahw < 0 else ahw)
    return dims, bnd, st


@pytest.mark.parametrize("name", CASES)
def test_partition_and_init_bit_exact(name):
    z = _load(name)
    dims, bnd, stages = _stages_for(z)
    assert np.array_equal(np.array(bnd), z["boundaries"])
    for j, st in enumerate(stages):
        flat = np.concatenate([p.ravel() for p in st.params()])
        assert np.array_equal(flat, z[f"init_{j}"])           # same PCG64 draws


@pytest.mark.parametrize("name", CASES)
def test_sequential_local_steps_match_reference(name):
    z = _load(name)
    dims, bnd, stages = _stages_for(z)
    steps = int(z["steps"])
    losses = np.zeros((len(stages), steps))
    for t in range(steps):
        h = z["xs"][t]
        for j, st in enumerate(stages):
            loss, h, _ = orc.local_step(st, h, z["ys"][t], total_steps=steps, **HYPER)
            losses[j, t] = loss
            if t == 0:
                np.testing.assert_allclose(h, z[f"xout0_{j}"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(losses, z["losses"], rtol=0, atol=1e-12)
    for j, st in enumerate(stages):
        flat = np.concatenate([p.ravel() for p in st.params()])
        mom = np.concatenate([v.ravel() for v in st.momenta])
        np.testing.assert_allclose(flat, z[f"final_{j}"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(mom, z[f"mom_{j}"], rtol=0, atol=1e-12)
        assert st.step_count == int(z[f"step_count_{j}"])


def test_threaded_reference_equals_sequential_oracle():
    """the reference's threaded PPLL == sequential schedule."""
    z = np.load(os.path.join(GOLDEN, "threaded_ppll.npz"))
    dims = (24, 20, 16, 12, 6)
    stages = orc.build_stages(dims, orc.partition(dims, 3), 2, 1, 3)
    batches = list(zip(z["xs"], z["ys"]))
    losses = orc.sequential_ppll(stages, batches, 0.05, 0.001, 20, 0.9, 1e-4)
    np.testing.assert_allclose(np.array(losses), z["losses"], rtol=0, atol=1e-12)
    for j, st in enumerate(stages):
        flat = np.concatenate([p.ravel() for p in st.params()])
        np.testing.assert_allclose(flat, z[f"final_{j}"], rtol=0, atol=1e-12)


def test_roundrobin_traces_bit_exact():
    with open(os.path.join(GOLDEN, "roundrobin_traces.json")) as f:
        traces = json.load(f)
    for t in traces:
        tr = orc.roundrobin_trace(t["s"], t["n"], t["M"])
        assert float(tr.rounds) == t["wall_time"]
        assert tr.batches_processed == t["batches_processed"]
        assert {str(k): v for k, v in sorted(tr.staleness.items())} == t["staleness"]
        assert tr.high_water == t["high_water"]


def test_full_m_config_losses():
    """(3072,1024,1024,1024,1024,10), s=4, B=128, 3 steps vs the reference."""
    z = np.load(os.path.join(GOLDEN, "full_m.npz"))
    dims = (3072, 1024, 1024, 1024, 1024, 10)
    bnd = orc.partition(dims, 4)
    assert np.array_equal(np.array(bnd), z["boundaries"])
    stages = orc.build_stages(dims, bnd, 2, 3, 42)
    rng = np.random.default_rng(0)
    xs = rng.standard_normal((3, 128, 3072))
    ys = rng.integers(0, 10, size=(3, 128))
    losses = orc.sequential_ppll(stages, list(zip(xs, ys)), 0.05, 0.001, 100, 0.9, 1e-4)
    np.testing.assert_allclose(np.array(losses), z["losses"], rtol=0, atol=1e-11)
    for j, st in enumerate(stages):
        flat = np.concatenate([p.ravel() for p in st.params()])
        np.testing.assert_allclose(flat[:256], z[f"head_{j}"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(flat.sum(), z[f"sum_{j}"], rtol=1e-10)


# --- the reference tests' own known answers (test_optim.py, test_tensor.py,
#     test_blocks.py, test_runtime.py) restated against the oracle -----------

def test_optimizer_kats():
    th, v = np.array([1.0]), np.zeros(1)
    orc.nesterov_update(th, v, np.array([0.5]), 0.1, 0.0, 0.0)      # test_optim.py:15-24
    assert np.allclose(th, [0.95])
    th, v = np.array([0.0]), np.zeros(1)
    orc.nesterov_update(th, v, np.array([1.0]), 1.0, 0.9, 0.0)      # :27-34
    assert np.allclose(v, [1.0]) and np.allclose(th, [-1.9])
    orc.nesterov_update(th, v, np.array([1.0]), 1.0, 0.9, 0.0)      # :47-56
    assert np.allclose(v, [1.9]) and np.allclose(th, [-4.61])
    th, v = np.array([10.0]), np.zeros(1)
    orc.nesterov_update(th, v, np.array([0.0]), 1.0, 0.0, 1e-4)     # :37-44
    assert np.allclose(th, [9.999])


def test_cosine_kats():
    assert orc.cosine_lr(0, 0.2, 0.02, 100) == pytest.approx(0.2)     # test_optim.py:106-111
    assert orc.cosine_lr(100, 0.2, 0.02, 100) == pytest.approx(0.02)
    assert orc.cosine_lr(50, 0.2, 0.02, 100) == pytest.approx(0.11)
    with pytest.raises(ValueError):
        orc.cosine_lr(101, 0.2, 0.02, 100)


def test_xent_kats():
    loss, _ = orc.softmax_xent(np.zeros((3, 4)), np.array([0, 1, 3]))  # test_tensor.py:90-93
    assert loss == pytest.approx(math.log(4))
    loss, g = orc.softmax_xent(np.array([[1e4, 0.0], [0.0, 1e4]]), np.array([0, 1]))
    assert np.isfinite(loss) and np.all(np.isfinite(g))                  # :101-104


def test_aux_depth_kats():
    assert orc.aux_depth(0, 4, 3) == 4                                   # test_blocks.py:90-94
    assert orc.aux_depth(3, 4, 3) == 3
    assert orc.aux_depth(11, 2, 3) == 0
    assert orc.aux_depth(1, 2, 3) == 2


def test_deterministic_trace_kat():
    tr = orc.roundrobin_trace(2, 4, 1)                                   # test_runtime.py:199-210
    assert tr.batches_processed == [4, 4]
    assert dict(tr.staleness) == {0: 8}
    assert tr.high_water == [1, 1]
    assert tr.rounds == 5


@pytest.mark.parametrize("tag", ["s2", "s4", "s3"])
def test_e2e_naive_pp_match_reference(tag):
    """E2E / naive-PP restatement vs the reference's four runs (threaded and
    deterministic, both modes; bitwise identical there)."""
    z = np.load(os.path.join(GOLDEN, "e2e_naive.npz"))
    dims = tuple(int(d) for d in z[f"{tag}_dims"])
    s = int(z[f"{tag}_s"])
    plan = orc.partition(dims, s)
    stages = orc.build_stages(dims, plan, 2, 3, 42)
    losses = [orc.e2e_step(stages, x, y, 0.05, 0.001, 10, 0.9, 1e-4)
              for x, y in zip(z[f"{tag}_xs"], z[f"{tag}_ys"])]
    np.testing.assert_allclose(losses, z[f"{tag}_losses"], rtol=0, atol=1e-12)
    assert list(z[f"{tag}_n_losses"]) == [0] * (s - 1) + [len(losses)]
    for j, st in enumerate(stages):
        f = np.concatenate([p.ravel() for p in st.params()])
        mv = np.concatenate([v.ravel() for v in st.momenta])
        np.testing.assert_allclose(f, z[f"{tag}_final_{j}"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(mv, z[f"{tag}_mom_{j}"], rtol=0, atol=1e-12)
        assert st.step_count == int(z[f"{tag}_step_{j}"])
