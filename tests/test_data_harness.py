"""Host-side data path and metrics CSV against the reference (no GPU):
BatchIterator orders (data.py:148-179) and the metrics CSV text
(harness.py:238-252) are pinned to fixtures the reference produced
(tests/golden/gen_golden.py: gen_data_and_csv)."""
import json
import os

import numpy as np
import pytest

import paper_2411_12780_b200 as lp
from conftest import GOLDEN


def test_batch_orders_match_reference():
    cases = json.load(open(os.path.join(GOLDEN, "batch_orders.json")))
    for c in cases:
        n = c["n"]
        ds = lp.Dataset(np.arange(n, dtype=np.float64)[:, None], np.zeros(n, dtype=np.int64), 1)
        it = lp.batches(ds, c["bs"], shuffle=c["shuffle"], seed=c["seed"])
        assert len(it) == c["len"]
        got = [[int(v) for v in f[:, 0]] for f, _ in it]
        assert got == c["batches"], c


def test_metrics_csv_matches_reference(tmp_path):
    recs = [lp.MetricsRecord("PPLL", 1, 12.5, 0.25, 0.5, 0.375, 1000, 2000, 0.125),
            lp.MetricsRecord("E2E", 0, 3.0, 2.302585093, 0.1, 0.09999999, 7, 8, 0.0),
            lp.MetricsRecord("PPLL", 0, 1e-7, 1.0 / 3.0, 1.0, 0.0, 0, 0, 1.5)]
    out = tmp_path / "m.csv"
    lp.write_metrics_csv(recs, out)
    assert out.read_text() == open(os.path.join(GOLDEN, "metrics_ref.csv")).read()
    with pytest.raises(lp.InvalidValue):
        lp.write_metrics_csv([], out)
    with pytest.raises(lp.IoError):
        lp.write_metrics_csv(recs, tmp_path / "missing-dir" / "m.csv")


def test_dataset_validation():
    f = np.zeros((4, 3))
    with pytest.raises(lp.InvalidArg):
        lp.Dataset(np.zeros((0, 3)), np.zeros(0, dtype=np.int64), 2)
    with pytest.raises(lp.InvalidArg):
        lp.Dataset(f, np.zeros(3, dtype=np.int64), 2)
    with pytest.raises(lp.InvalidArg):
        lp.Dataset(f, np.array([0, 1, 2, 0]), 2)
    bad = f.copy()
    bad[0, 0] = np.nan
    with pytest.raises(lp.InvalidArg):
        lp.Dataset(bad, np.zeros(4, dtype=np.int64), 2)
    with pytest.raises(lp.InvalidArg):
        lp.batches(lp.Dataset(f, np.zeros(4, dtype=np.int64), 1), 0)
    ds = lp.Dataset(f, np.zeros(4, dtype=np.int64), 1)
    assert (ds.n, ds.dim) == (4, 3)


# ---- dataset sources (data.py:52-144), pinned to the reference's outputs ----

def _ds_golden():
    return np.load(os.path.join(GOLDEN, "datasets.npz"))


def test_gen_blobs_bitwise_equal_reference():
    g = _ds_golden()
    for i in range(5):
        npc, c, d, spread, seed = g[f"blobs{i}_args"]
        ds = lp.gen_blobs(int(npc), int(c), int(d), float(spread), int(seed))
        assert ds.features.dtype == np.float64 and ds.num_classes == int(c)
        assert np.array_equal(ds.features, g[f"blobs{i}_x"]), i
        assert np.array_equal(ds.labels, g[f"blobs{i}_y"]), i


def test_gen_spirals_bitwise_equal_reference():
    g = _ds_golden()
    for i in range(3):
        npc, noise, seed = g[f"spiral{i}_args"]
        ds = lp.gen_spirals(int(npc), float(noise), int(seed))
        assert np.array_equal(ds.features, g[f"spiral{i}_x"]), i
        assert np.array_equal(ds.labels, g[f"spiral{i}_y"]), i
    a0, a1 = lp.spiral_reference(200)
    assert np.array_equal(a0, g["spiral_ref0"]) and np.array_equal(a1, g["spiral_ref1"])


def test_generator_argument_checks():
    for args in ((0, 2, 2, 0.5, 0), (5, 2, 0, 0.5, 0), (5, 0, 2, 0.5, 0), (5, 2, 2, -0.1, 0)):
        with pytest.raises(lp.InvalidArg):
            lp.gen_blobs(*args)
    for args in ((0, 0.1, 0), (10, -0.1, 0)):
        with pytest.raises(lp.InvalidArg):
            lp.gen_spirals(*args)


def _write(tmp_path, name, data):
    p = tmp_path / name
    p.write_bytes(bytes(data))
    return p


def test_load_idx_equals_reference(tmp_path):
    g = _ds_golden()
    ip = _write(tmp_path, "i.idx", g["idx_images"])
    lp_ = _write(tmp_path, "l.idx", g["idx_labels"])
    ds = lp.load_idx(ip, lp_)
    assert np.array_equal(ds.features, g["idx_x"]) and np.array_equal(ds.labels, g["idx_y"])
    assert ds.num_classes == int(g["idx_classes"])
    assert ds.pixels.dtype == np.uint8 and np.array_equal(ds.pixels / 255.0, ds.features)


def test_load_idx_errors(tmp_path):
    import struct
    img = struct.pack(">IIII", 0x803, 2, 2, 2) + bytes(range(8))
    lbl = struct.pack(">II", 0x801, 2) + bytes([0, 1])
    ok_i, ok_l = _write(tmp_path, "i", img), _write(tmp_path, "l", lbl)
    assert lp.load_idx(ok_i, ok_l).n == 2
    with pytest.raises(lp.BadMagic):
        lp.load_idx(_write(tmp_path, "bi", struct.pack(">I", 0x801) + img[4:]), ok_l)
    with pytest.raises(lp.BadMagic):
        lp.load_idx(ok_i, _write(tmp_path, "bl", struct.pack(">I", 0x803) + lbl[4:]))
    with pytest.raises(lp.CountMismatch):
        lp.load_idx(ok_i, _write(tmp_path, "cl", struct.pack(">II", 0x801, 3) + bytes([0, 1, 0])))
    with pytest.raises(lp.TruncatedFile):
        lp.load_idx(_write(tmp_path, "ti", img[:-1]), ok_l)
    with pytest.raises(lp.TruncatedFile):
        lp.load_idx(_write(tmp_path, "th", img[:10]), ok_l)
    with pytest.raises(lp.TruncatedFile):
        lp.load_idx(ok_i, _write(tmp_path, "tl", lbl[:-1]))
    assert issubclass(lp.TruncatedFile, lp.LocopipeError)


def test_experiment_config_validation():
    ok = dict(dataset="blobs", layer_dims=(2, 8, 2))
    lp.ExperimentConfig(**ok)
    for bad in (dict(dataset="cifar"), dict(layer_dims=(4,)), dict(layer_dims=(4, 0, 2)),
                dict(stages=3), dict(batch_size=0), dict(momentum=1.0), dict(lr0=0.01, lr_min=0.1),
                dict(spread=-1.0), dict(aux_hidden_width=0), dict(sleep_padding=(-1.0,)),
                dict(modes=()), dict(modes=(lp.RunMode.PPLL, lp.RunMode.PPLL)),
                dict(dataset="idx"), dict(precision="fp16")):
        with pytest.raises(lp.InvalidValue):
            lp.ExperimentConfig(**{**ok, **bad})


def test_make_datasets_checks_widths():
    train, test = lp.make_datasets(lp.ExperimentConfig(dataset="blobs", classes=3, dim=4,
                                                       layer_dims=(4, 8, 3), seed=5))
    assert np.array_equal(train.features, lp.gen_blobs(100, 3, 4, 0.5, 5).features)
    assert np.array_equal(test.features, lp.gen_blobs(100, 3, 4, 0.5, 6).features)
    with pytest.raises(lp.ConfigMismatch):
        lp.make_datasets(lp.ExperimentConfig(dataset="blobs", layer_dims=(3, 8, 2)))
    with pytest.raises(lp.ConfigMismatch):
        lp.make_datasets(lp.ExperimentConfig(dataset="spirals", layer_dims=(2, 8, 3)))


def test_report_table_layout():
    rep = lp.ComparisonReport(2, 0.5, 0.75, (lp.ModeSummary("E2E", 1.5, 0.25, 10, 20),
                                             lp.ModeSummary("PPLL", 12.0, 0.5, 1000, 2)), 2.0)
    assert lp.report_table(rep) == (
        "mode  batches_per_sec  test_acc  params_max_stage  activations_max_stage\n"
        "E2E   1.500000         0.250000  10                20\n"
        "PPLL  12.000000        0.500000  1000              2\n"
        "analytic (k+1)/s = 0.750000\n")
