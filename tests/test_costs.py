"""Batch-time model and schedule simulator vs the reference (costs.py):
analytic forms, per-event timelines, makespans, steady batch times and the
Gantt CSV are pinned to values the reference produced (tests/golden/
gen_golden.py: gen_costs) — bit-exact, the arithmetic order is the same."""
import json
import os

import pytest

import paper_2411_12780_b200 as lp
from conftest import GOLDEN

G = json.load(open(os.path.join(GOLDEN, "costs.json")))


@pytest.mark.parametrize("ci", range(len(G["cases"])))
def test_costs_match_reference(ci):
    c = G["cases"][ci]
    sp = [lp.StageProfile(*p) for p in c["profiles"]]
    cm = lp.CommModel(c["q"])
    for name, fn in (("t_e2e", lambda: lp.t_e2e(sp)), ("t_pp", lambda: lp.t_pp(sp, cm)),
                     ("t_ppll", lambda: lp.t_ppll(sp, cm))):
        est = fn()
        assert est.batch_time == c[name][0]
        assert est.components == c[name][1]
    beats, margins = lp.ppll_beats_pp(sp, cm)
    assert [beats, margins] == c["beats"]
    for key, want in c["sims"].items():
        mode, n, cap = key.split("/")
        r = lp.simulate_schedule(sp, cm, mode, int(n), int(cap))
        assert r.makespan == want["makespan"] and r.steady_batch_time == want["steady"]
        assert list(r.batch_finish) == want["finish"]
        assert [[e.stage, e.kind, e.batch_id, e.start, e.end] for e in r.events] == want["events"]
    assert lp.render_gantt_csv(lp.simulate_schedule(sp, cm, "ppll", 4, 2).events) == c["gantt"]


def test_ratio_ideal_and_errors():
    for k, s, want in G["ratios"]:
        assert lp.ratio_ideal(k, s) == want
    with pytest.raises(ValueError):
        lp.ratio_ideal(-1.0, 2)
    with pytest.raises(ValueError):
        lp.ratio_ideal(0.5, 0)
    with pytest.raises(lp.EmptyProfiles):
        lp.t_e2e([])
    with pytest.raises(lp.InvalidMode):
        lp.simulate_schedule([lp.StageProfile(1, 1, 1)], lp.CommModel(), "bogus", 3)
    with pytest.raises(lp.EmptyEvents):
        lp.render_gantt_csv([])
    with pytest.raises(ValueError):
        lp.StageProfile(-1.0, 0, 0)
    with pytest.raises(lp.ZeroDuration):
        lp.steady_throughput(lp.simulate_schedule([lp.StageProfile(0, 0, 0)], lp.CommModel(),
                                                  "ppll", 3))


def test_idle_fraction_of_balanced_and_skewed_pipelines():
    bal = [lp.StageProfile(1.0, 2.0, 0.0)] * 4
    r = lp.simulate_schedule(bal, lp.CommModel(), "ppll", 40, 2)
    assert r.steady_batch_time == pytest.approx(3.0)
    assert max(r.idle_fraction(4)) < 1e-9
    skew = [lp.StageProfile(1.0, 2.0, 0.0)] * 3 + [lp.StageProfile(1.0, 1.0, 0.0)]
    r = lp.simulate_schedule(skew, lp.CommModel(), "ppll", 40, 2)
    idle = r.idle_fraction(4)
    assert idle[3] == pytest.approx(1.0 / 3.0, abs=1e-9) and max(idle[:3]) < 1e-9
