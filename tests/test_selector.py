"""Context-aware strategy selection: the alpha + beta * rows fit
(SPEC CostParams), the decision table / split threshold,
and the engine resolving a calibrated `auto` table per batch with no timing
(planned on the device-free dry path)."""
import json

import pytest

from paper_2605_21603_b200 import opflow as of
from paper_2605_21603_b200 import selector as sl
from util import unit_costs

R = of.PartitionRule
SEQ = {"name": "sequential"}
SPLIT = {"name": "split_overlap"}
DBO3 = {"name": "split_overlap", "n_ubatches": 3}


def test_fit_line_recovers_affine_and_clamps():
    r = [256, 1024, 4096, 8192]
    a, b = sl.fit_line(r, [0.3 + 0.002 * x for x in r])
    assert a == pytest.approx(0.3) and b == pytest.approx(0.002)
    # noisy, would fit a negative intercept -> refit through the origin
    a, b = sl.fit_line([100, 200], [0.9, 2.0])
    assert a == 0.0 and b == pytest.approx((100 * 0.9 + 200 * 2.0) / (100 ** 2 + 200 ** 2))
    # decreasing times -> rows-independent
    a, b = sl.fit_line([100, 200], [2.0, 1.0])
    assert (a, b) == (1.5, 0.0)
    assert sl.fit_line([64], [0.64]) == (0.0, pytest.approx(0.01))
    with pytest.raises(ValueError):
        sl.fit_line([], [])


def _selector(lines, margin=0.0, cands=(SEQ, SPLIT)):
    s = sl.StrategySelector(list(cands), margin=margin)
    for c, (a, b) in zip(cands, lines):
        for r in (128, 1024, 8192):
            s.add(c, r, a + b * r)
    return s.fit()


def test_split_threshold_is_the_crossover():
    # sequential: 0.1 + 0.010 r ; split: 0.5 + 0.009 r  -> crossover at 400 rows
    s = _selector([(0.1, 0.010), (0.5, 0.009)])
    assert s.choose(100) == SEQ and s.choose(399) == SEQ
    assert s.choose(401) == SPLIT and s.choose(100000) == SPLIT
    t = s.table()
    assert [e["min_rows"] for e in t] == [0, 401] or [e["min_rows"] for e in t] == [0, 400]
    assert t[0]["strategy"] == SEQ and t[-1]["strategy"] == SPLIT
    # the table is exactly the argmin everywhere
    for r in range(0, 2000, 7):
        pick = [e for e in t if e["min_rows"] <= r][-1]["strategy"]
        best = min((SEQ, SPLIT), key=lambda c: s.predict(c, r))
        if abs(s.predict(SEQ, r) - s.predict(SPLIT, r)) > 1e-9:
            assert pick == best, r


def test_margin_moves_the_threshold_toward_sequential():
    s0 = _selector([(0.1, 0.010), (0.5, 0.009)])
    s5 = _selector([(0.1, 0.010), (0.5, 0.009)], margin=0.05)
    assert s5.thresholds()[0] > s0.thresholds()[0]
    # a challenger that is never 5% better is never chosen
    s = _selector([(0.1, 0.010), (0.1, 0.0099)], margin=0.05)
    assert s.table() == [{"min_rows": 0, "strategy": SEQ}]


def test_three_candidates_lower_envelope():
    s = _selector([(0.0, 0.010), (0.4, 0.009), (1.6, 0.0085)], cands=(SEQ, SPLIT, DBO3))
    t = s.table()
    assert [e["strategy"] for e in t] == [SEQ, SPLIT, DBO3]
    for r in range(0, 6000, 13):
        pick = [e for e in t if e["min_rows"] <= r][-1]["strategy"]
        vals = sorted(s.predict(c, r) for c in (SEQ, SPLIT, DBO3))
        assert s.predict(pick, r) <= vals[0] + 1e-9
    rep = s.report()
    assert len(rep["lines_ms"]) == 3 and rep["table"] == t
    json.dumps(rep)


def test_selector_errors():
    with pytest.raises(ValueError):
        sl.StrategySelector([])
    with pytest.raises(ValueError):
        sl.StrategySelector([SEQ], margin=1.0)
    s = sl.StrategySelector([SEQ, SPLIT])
    with pytest.raises(KeyError):
        s.add({"name": "dbo"}, 10, 1.0)
    s.add(SEQ, 10, 1.0)
    with pytest.raises(ValueError):
        s.fit()  # SPLIT has no timings


@pytest.mark.usefixtures("built")
def test_engine_resolves_calibrated_table_per_rows():
    desc = of.dense_tp_graph(2, 1024, 64, dtype="f32", costs=unit_costs())
    g = of.build_graph(desc)
    p = of.partition(g, [R.by_func("AllReduce")])
    spec = {"name": "auto", "table": [{"min_rows": 0, "strategy": SEQ},
                                      {"min_rows": 512, "strategy": {"name": "split_overlap", "sizes": None}}]}
    spec["table"][1]["strategy"] = {"name": "split_overlap"}
    for rows, want in [(64, SEQ), (511, SEQ), (512, SPLIT), (1024, SPLIT)]:
        got, st = of.dry_run(g, p, spec, rows=rows)
        ref, _ = of.dry_run(g, p, want, rows=rows)
        assert [(d["subgraphs"], d["lane"], d["rows"]) for d in got["dispatches"]] == \
               [(d["subgraphs"], d["lane"], d["rows"]) for d in ref["dispatches"]], rows
        assert st["auto"][0]["chosen"] == json.dumps(want, separators=(",", ":"))


@pytest.mark.usefixtures("built")
def test_engine_table_errors():
    g = of.build_graph(of.dense_tp_graph(1, 8, 4, costs=unit_costs()))
    p = of.partition(g, [])
    bad = [{"name": "auto", "table": []},
           {"name": "auto", "table": [{"min_rows": 4, "strategy": SEQ}]},  # nothing for rows < 4
           {"name": "auto", "table": [{"min_rows": 0}]},
           {"name": "auto", "candidates": [SEQ]}]  # timed selection needs a device
    codes = []
    for spec in bad:
        with pytest.raises(of.Error) as e:
            of.dry_run(g, p, spec, rows=2)
        codes.append(e.value.code)
    assert codes[:3] == [of.ERRC.index("ConfigError")] * 3
    assert codes[3] == of.ERRC.index("EngineStopped")


def test_op_costs_from_trace_and_apply():
    pts = {}
    for r in (256, 1024, 4096):
        tr = [{"name": "l0.qkv u0", "dur": 5.0 + 0.01 * r}, {"name": "l0.attn u0", "dur": 0.002 * r},
              {"name": "l0.attn u1", "dur": 0.002 * r}, {"name": "l0.norm u0", "dur": 3.0}]
        pts[r] = sl.op_times_from_trace(tr)
    assert pts[1024]["l0.attn"] == pytest.approx(2 * 0.002 * 1024 * 1e-3)
    c = sl.fit_op_costs(pts)
    assert c["l0.qkv"] == (pytest.approx(5.0), pytest.approx(0.01))
    assert c["l0.attn"][0] == pytest.approx(0.0, abs=1e-9) and c["l0.attn"][1] == pytest.approx(0.004)
    assert c["l0.norm"] == (pytest.approx(3.0), pytest.approx(0.0, abs=1e-12))
    # measured costs feed partition's dominant class (SURVEY Appendix A:
    # filler#2 = {layer0.norm, layer1.attn, layer1.mlp} is memory-dominant at
    # unit costs, B=4; a measured-heavy layer1.mlp makes it compute-dominant)
    desc = of.dense_tp_graph(2, 4, 4, costs=unit_costs())
    rules = [R.by_func("AllReduce")]
    assert of.partition(of.build_graph(desc), rules).subgraphs[2].dominant_class == of.ResourceClass.kMemory
    out = sl.apply_op_costs(desc, {"layer1.mlp": (100.0, 10.0), "layer0.norm": (1.0, 0.05)})
    ops = {o["name"]: o for o in json.loads(out)["operators"]}
    assert ops["layer1.mlp"]["cost"] == [100.0, 10.0]
    assert ops["layer1.attn"]["cost"] == [0.0, 0.0]  # no launch of its own in the measurement
    p2 = of.partition(of.build_graph(out), rules)
    assert p2.subgraphs[2].dominant_class == of.ResourceClass.kCompute
    assert [s_.label for s_ in p2.subgraphs] == [s_.label for s_ in of.partition(of.build_graph(desc), rules).subgraphs]
    gd = sl.apply_op_costs(of.GraphDescription.from_json(desc), {"layer1.mlp": (3.0, 0.5)})
    assert [o.cost for o in gd.operators if o.name == "layer1.mlp"][0] == of.CostParams(3.0, 0.5)
