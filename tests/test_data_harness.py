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
