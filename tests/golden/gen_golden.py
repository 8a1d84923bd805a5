"""Generate golden vectors for the PPLL hot path FROM THE REFERENCE ITSELF.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_golden.py

It imports ``locopipe`` from ``/root/reference/pkg/src`` and drives its public
API (``build_modules``, ``local_loss_and_update``, ``run_deterministic``,
``run_epoch``) on fixed seeds, then writes small ``.npz`` fixtures next to this
script.  Nothing at test time reads /root/reference: the fixtures travel.
"""
from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import locopipe as lp  # noqa: E402

# (name, dims, s, d_prime, interval, seed, batch, steps, aux_hidden_width)
CASES = [
    ("mlp_s1", (48, 32, 10), 1, 0, 1, 7, 8, 4, None),
    ("mlp_s2", (48, 40, 32, 24, 10), 2, 2, 3, 42, 16, 5, None),
    ("mlp_s4", (96, 64, 64, 48, 40, 10), 4, 2, 3, 42, 16, 5, None),
    ("mlp_s3_wide_aux", (40, 36, 28, 20, 10), 3, 1, 1, 5, 12, 4, 24),
    ("mlp_s4_odd", (33, 17, 29, 13, 21, 7), 4, 3, 2, 11, 9, 6, None),
]

HYPER = dict(lr0=0.05, lr_min=0.001, momentum=0.9, weight_decay=1e-4)


def make(dims, s, d_prime, interval, seed, total_steps, aux_hidden_width):
    spec = lp.NetworkSpec(tuple(dims))
    plan = lp.partition(spec, s)
    hyper = lp.Hyperparams(total_steps=total_steps, seed=seed,
                           aux_hidden_width=aux_hidden_width, **HYPER)
    return plan, lp.build_modules(spec, plan, d_prime, interval, hyper)


def flat(mod):
    return np.concatenate([p.data.ravel() for p in mod.parameters()])


def flat_m(mod):
    return np.concatenate([mod.optimizer.buffer_for(p).ravel()
                           for p in mod.parameters()])


def gen_case(name, dims, s, d_prime, interval, seed, B, steps, ahw):
    plan, mods = make(dims, s, d_prime, interval, seed, steps, ahw)
    rng = np.random.default_rng(1000 + seed)
    xs = rng.standard_normal((steps, B, dims[0]))
    ys = rng.integers(0, dims[-1], size=(steps, B))
    out = {
        "dims": np.array(dims), "s": s, "d_prime": d_prime, "interval": interval,
        "seed": seed, "batch": B, "steps": steps,
        "aux_hidden_width": -1 if ahw is None else ahw,
        "boundaries": np.array(plan.boundaries),
        "assigned_aux_depth": np.array([m.assigned_aux_depth for m in mods]),
        "xs": xs, "ys": ys,
    }
    for j, m in enumerate(mods):
        out[f"init_{j}"] = flat(m)
        out[f"shapes_{j}"] = np.array([list(p.shape) + [0] * (2 - len(p.shape))
                                       for p in m.parameters()])
    losses = np.zeros((s, steps))
    for t in range(steps):
        h = lp.Tensor(xs[t])
        for j, m in enumerate(mods):
            loss, h = lp.local_loss_and_update(m, h, ys[t])
            losses[j, t] = loss
            if t == 0:
                out[f"xout0_{j}"] = h.data.copy()
        # logits of the final stage after the step are not needed; x_out is
    out["losses"] = losses
    for j, m in enumerate(mods):
        out[f"final_{j}"] = flat(m)
        out[f"mom_{j}"] = flat_m(m)
        out[f"step_count_{j}"] = m.optimizer.step_count
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    return losses


def gen_threaded_equivalence():
    """threaded PPLL (run_epoch) == sequential loop, on the reference."""
    dims = (24, 20, 16, 12, 6)
    data_rng = np.random.default_rng(5)
    data = [(data_rng.standard_normal((6, 24)), data_rng.integers(0, 6, 6))
            for _ in range(7)]
    _, mods = make(dims, 3, 2, 1, 3, 20, None)
    m = lp.run_epoch(lp.RunMode.PPLL, mods, iter(data), lp.RunConfig(buffer_capacity=2))
    out = {"xs": np.stack([d[0] for d in data]), "ys": np.stack([d[1] for d in data]),
           "losses": np.array(m.loss_history)}
    for j, mod in enumerate(mods):
        out[f"final_{j}"] = flat(mod)
    np.savez_compressed(os.path.join(HERE, "threaded_ppll.npz"), **out)


def gen_traces():
    """Deterministic round-robin integer bookkeeping (runtime.py:475-533)."""
    traces = []
    for s, n, M in [(2, 4, 1), (2, 7, 2), (3, 5, 1), (3, 9, 3), (4, 6, 2),
                    (4, 1, 1), (5, 12, 2), (1, 5, 2), (4, 0, 2)]:
        dims = (4,) + (5,) * s + (2,)
        _, mods = make(dims, s, 1, 1, 0, 64, None)
        rng = np.random.default_rng(s * 100 + n)
        data = [(rng.standard_normal((3, 4)), rng.integers(0, 2, 3)) for _ in range(n)]
        m = lp.run_deterministic(lp.RunMode.PPLL, mods, iter(data),
                                 lp.RunConfig(buffer_capacity=M))
        traces.append({
            "s": s, "n": n, "M": M, "wall_time": m.wall_time,
            "busy_time": m.busy_time, "batches_processed": m.batches_processed,
            "staleness": {str(k): v for k, v in sorted(m.staleness.items())},
            "high_water": m.buffer_high_water, "n_batches": m.n_batches,
        })
    with open(os.path.join(HERE, "roundrobin_traces.json"), "w") as f:
        json.dump(traces, f, indent=1, sort_keys=True)


def gen_full_m():
    """The CIFAR-shaped MLP analog (SURVEY §8 'M'): losses + param checksums."""
    dims = (3072, 1024, 1024, 1024, 1024, 10)
    steps, B = 3, 128
    plan, mods = make(dims, 4, 2, 3, 42, 100, None)
    rng = np.random.default_rng(0)
    xs = rng.standard_normal((steps, B, 3072))
    ys = rng.integers(0, 10, size=(steps, B))
    losses = np.zeros((4, steps))
    for t in range(steps):
        h = lp.Tensor(xs[t])
        for j, m in enumerate(mods):
            loss, h = lp.local_loss_and_update(m, h, ys[t])
            losses[j, t] = loss
    out = {"losses": losses, "data_seed": 0, "steps": steps, "batch": B,
           "boundaries": np.array(plan.boundaries)}
    for j, m in enumerate(mods):
        f = flat(m)
        out[f"sum_{j}"] = f.sum()
        out[f"abssum_{j}"] = np.abs(f).sum()
        out[f"sq_{j}"] = (f * f).sum()
        out[f"head_{j}"] = f[:256]
        out[f"tail_{j}"] = f[-256:]
    np.savez_compressed(os.path.join(HERE, "full_m.npz"), **out)


def gen_e2e_naive():
    """The paper's baselines on the reference: end-to-end backprop (E2E) and
    naive pipeline parallelism (NAIVE_PP), threaded and deterministic.  All
    four runs are bitwise identical on the reference (test_runtime.py:154-194);
    the fixture keeps one copy plus the per-run agreement flags."""
    out = {}
    for tag, dims, s in [("s2", (48, 40, 32, 24, 10), 2), ("s4", (96, 64, 64, 48, 40, 10), 4),
                         ("s3", (33, 17, 29, 13, 21, 7), 3)]:
        rng = np.random.default_rng(77 + s)
        B, n = 12, 5
        data = [(rng.standard_normal((B, dims[0])), rng.integers(0, dims[-1], B))
                for _ in range(n)]
        runs = []
        for mode in (lp.RunMode.E2E, lp.RunMode.NAIVE_PP):
            for runner in (lp.run_deterministic, lp.run_epoch):
                _, mods = make(dims, s, 2, 3, 42, 10, None)
                m = runner(mode, mods, iter(data), lp.RunConfig(buffer_capacity=2))
                runs.append((m, mods))
        m0, mods0 = runs[0]
        same = all(np.array_equal(flat(a), flat(b)) for _, ms in runs[1:]
                   for a, b in zip(mods0, ms))
        same_loss = all(m.loss_history == m0.loss_history for m, _ in runs[1:])
        assert same and same_loss, tag
        out[f"{tag}_dims"] = np.array(dims)
        out[f"{tag}_s"] = s
        out[f"{tag}_xs"] = np.stack([d[0] for d in data])
        out[f"{tag}_ys"] = np.stack([d[1] for d in data])
        out[f"{tag}_losses"] = np.array(m0.loss_history[s - 1])
        out[f"{tag}_n_losses"] = np.array([len(h) for h in m0.loss_history])
        for j, mod in enumerate(mods0):
            out[f"{tag}_final_{j}"] = flat(mod)
            out[f"{tag}_mom_{j}"] = flat_m(mod)
            out[f"{tag}_step_{j}"] = mod.optimizer.step_count
    np.savez_compressed(os.path.join(HERE, "e2e_naive.npz"), **out)


def gen_data_and_csv():
    """BatchIterator orders (data.py:148-179) and the metrics CSV text
    (harness.py:238-252) from the reference."""
    orders = []
    for n, bs, shuffle, seed in [(10, 3, True, 0), (10, 3, False, 0), (7, 7, True, 5),
                                 (13, 4, True, 123), (1, 2, True, 9), (64, 16, True, 42)]:
        ds = lp.Dataset(np.arange(n, dtype=np.float64)[:, None], np.zeros(n, dtype=np.int64), 1)
        it = lp.batches(ds, bs, shuffle=shuffle, seed=seed)
        orders.append({"n": n, "bs": bs, "shuffle": shuffle, "seed": seed, "len": len(it),
                       "batches": [[int(v) for v in f[:, 0]] for f, _ in it]})
    recs = [lp.MetricsRecord("PPLL", 1, 12.5, 0.25, 0.5, 0.375, 1000, 2000, 0.125),
            lp.MetricsRecord("E2E", 0, 3.0, 2.302585093, 0.1, 0.09999999, 7, 8, 0.0),
            lp.MetricsRecord("PPLL", 0, 1e-7, 1.0 / 3.0, 1.0, 0.0, 0, 0, 1.5)]
    path = os.path.join(HERE, "metrics_ref.csv")
    lp.write_metrics_csv(recs, path)
    with open(os.path.join(HERE, "batch_orders.json"), "w") as f:
        json.dump(orders, f, indent=0)


def gen_datasets():
    """Synthetic generators (data.py:52-104) and the IDX reader (data.py:107-144)
    of the reference on fixed seeds / hand-packed bytes."""
    import tempfile
    out = {}
    for i, (npc, c, d, spread, seed) in enumerate([(30, 3, 5, 0.4, 1), (2, 4, 2, 0.0, 0),
                                                    (10, 2, 3, 0.5, 7), (7, 9, 2, 0.25, 11),
                                                    (4, 5, 1, 1.5, 3)]):
        ds = lp.gen_blobs(npc, c, d, spread, seed)
        out[f"blobs{i}_args"] = np.array([npc, c, d, spread, seed], dtype=np.float64)
        out[f"blobs{i}_x"], out[f"blobs{i}_y"] = ds.features, ds.labels
    for i, (npc, noise, seed) in enumerate([(150, 0.0, 4), (150, 0.05, 4), (33, 0.2, 9)]):
        ds = lp.gen_spirals(npc, noise, seed)
        out[f"spiral{i}_args"] = np.array([npc, noise, seed], dtype=np.float64)
        out[f"spiral{i}_x"], out[f"spiral{i}_y"] = ds.features, ds.labels
    a0, a1 = lp.spiral_reference(200)
    out["spiral_ref0"], out["spiral_ref1"] = a0, a1
    rng = np.random.default_rng(77)
    count, rows, cols = 37, 5, 7
    img = struct.pack(">IIII", 0x803, count, rows, cols) + \
        rng.integers(0, 256, count * rows * cols, dtype=np.uint8).tobytes() + b"tail"
    lbl = struct.pack(">II", 0x801, count) + rng.integers(0, 6, count, dtype=np.uint8).tobytes()
    with tempfile.TemporaryDirectory() as td:
        ip, lp_ = os.path.join(td, "i.idx"), os.path.join(td, "l.idx")
        open(ip, "wb").write(img)
        open(lp_, "wb").write(lbl)
        ds = lp.load_idx(ip, lp_)
    out["idx_images"] = np.frombuffer(img, dtype=np.uint8)
    out["idx_labels"] = np.frombuffer(lbl, dtype=np.uint8)
    out["idx_x"], out["idx_y"] = ds.features, ds.labels
    out["idx_classes"] = np.array(ds.num_classes)
    np.savez_compressed(os.path.join(HERE, "datasets.npz"), **out)


def gen_experiment():
    """harness.run_experiment (deterministic) on blobs and spirals configs:
    every metrics column except batches/s, plus the report's shape."""
    from locopipe.config import ExperimentConfig
    out = []
    for kw in [dict(dataset="blobs", n_per_class=40, classes=4, dim=6, spread=0.6, seed=3,
                    layer_dims=(6, 24, 20, 16, 4), stages=3, batch_size=16, epochs=2,
                    lr0=0.05, lr_min=0.001, aux_depth_max=1, aux_depth_interval=2),
               dict(dataset="spirals", n_per_class=50, noise=0.05, seed=9,
                    layer_dims=(2, 32, 32, 2), stages=2, batch_size=20, epochs=2, lr0=0.1)]:
        cfg = ExperimentConfig(**kw)
        recs, rep = lp.run_experiment(cfg, deterministic=True)
        out.append({"config": {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()},
                    "records": [[r.mode, r.epoch, r.mean_loss, r.train_acc, r.test_acc,
                                 r.params_max_stage, r.activations_max_stage, r.mean_staleness]
                                for r in recs],
                    "modes": [sm.mode for sm in rep.summaries], "stages": rep.stages})
    with open(os.path.join(HERE, "experiment.json"), "w") as f:
        json.dump(out, f, indent=0)


def gen_experiment_idx():
    """run_experiment on an IDX image/label pair (data.py:118-144 through
    harness.py:78-206), deterministic schedule, all three modes."""
    import tempfile
    from locopipe.config import ExperimentConfig
    rng = np.random.default_rng(21)
    count, rows, cols = 90, 4, 5
    lab = rng.integers(0, 3, count).astype(np.uint8)
    # class-dependent pixel means so the run learns something
    pix = np.clip(rng.normal(60 + 60 * lab[:, None], 40, (count, rows * cols)), 0, 255).astype(np.uint8)
    img = struct.pack(">IIII", 0x803, count, rows, cols) + pix.tobytes()
    lbl = struct.pack(">II", 0x801, count) + lab.tobytes()
    with tempfile.TemporaryDirectory() as td:
        ip, lp_ = os.path.join(td, "i.idx"), os.path.join(td, "l.idx")
        open(ip, "wb").write(img)
        open(lp_, "wb").write(lbl)
        kw = dict(dataset="idx", idx_train_images=ip, idx_train_labels=lp_,
                  layer_dims=(rows * cols, 16, 12, 3), stages=2, batch_size=16, epochs=2,
                  lr0=0.05, lr_min=0.001, seed=5)
        recs, rep = lp.run_experiment(ExperimentConfig(**kw), deterministic=True)
    out = {"images": list(img), "labels": list(lbl),
           "config": {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()
                      if not k.startswith("idx_")},
           "records": [[r.mode, r.epoch, r.mean_loss, r.train_acc, r.test_acc,
                        r.params_max_stage, r.activations_max_stage, r.mean_staleness]
                       for r in recs]}
    with open(os.path.join(HERE, "experiment_idx.json"), "w") as f:
        json.dump(out, f)


def gen_costs():
    """costs.py analytic forms, simulator timelines and Gantt CSV (reference)."""
    cases = []
    profs = [
        [(1.0, 2.0, 0.5, 0.5, 1.0, 0.25), (1.0, 2.0, 0.5, 0.25, 0.5, 0.125),
         (1.0, 2.0, 0.5, 0.0, 0.0, 0.0)],
        [(0.3, 0.7, 0.1, 0.9, 1.1, 0.2), (0.5, 0.2, 0.05, 0.0, 0.0, 0.0)],
        [(2.0, 4.0, 1.0, 0.0, 0.0, 0.0)],
        [(0.1 * (j + 1), 0.3, 0.05, 0.2 / (j + 1), 0.1, 0.01) for j in range(5)],
    ]
    for pi, pr in enumerate(profs):
        sp = [lp.StageProfile(*p) for p in pr]
        for q in (0.0, 0.35):
            cm = lp.CommModel(q)
            case = {"profiles": pr, "q": q,
                    "t_e2e": [lp.t_e2e(sp).batch_time, lp.t_e2e(sp).components],
                    "t_pp": [lp.t_pp(sp, cm).batch_time, lp.t_pp(sp, cm).components],
                    "t_ppll": [lp.t_ppll(sp, cm).batch_time, lp.t_ppll(sp, cm).components],
                    "beats": list(lp.ppll_beats_pp(sp, cm)), "sims": {}}
            for mode in ("e2e", "naive_pp", "ppll"):
                for n, cap in ((7, 2), (3, 1), (12, 3)):
                    r = lp.simulate_schedule(sp, cm, mode, n, cap)
                    case["sims"][f"{mode}/{n}/{cap}"] = {
                        "makespan": r.makespan, "steady": r.steady_batch_time,
                        "finish": list(r.batch_finish),
                        "events": [[e.stage, e.kind, e.batch_id, e.start, e.end]
                                   for e in r.events]}
            case["gantt"] = lp.render_gantt_csv(
                lp.simulate_schedule(sp, cm, "ppll", 4, 2).events)
            cases.append(case)
    ratios = [[k, s, lp.ratio_ideal(k, s)] for k in (0.0, 0.5, 2.0) for s in (1, 2, 4, 8)]
    with open(os.path.join(HERE, "costs.json"), "w") as f:
        json.dump({"cases": cases, "ratios": ratios}, f)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[name]()
        print("ok")
        sys.exit(0)
    for case in CASES:
        print(case[0], gen_case(*case)[:, -1])
    gen_threaded_equivalence()
    gen_traces()
    gen_full_m()
    gen_e2e_naive()
    gen_data_and_csv()
    gen_costs()
    gen_datasets()
    gen_experiment()
    gen_experiment_idx()
    print("ok")
