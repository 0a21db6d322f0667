"""GPU: calibrated context-aware strategy selection on a real
engine — device-timed candidates at several batch sizes (row-prefix views of
max-size buffers), the fitted decision table replayed by the engine with no
timing, and per-op alpha/beta from the per-launch trace."""
import numpy as np
import pytest

from oracle import oracle
from paper_2605_21603_b200 import opflow as of
from paper_2605_21603_b200 import selector as sl
from paper_2605_21603_b200.workloads import llama_inputs, rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("built")]

SEQ = {"name": "sequential"}
SPLIT = {"name": "split_overlap", "align": 128}
MAX_ROWS = 1024


def _setup():
    import torch
    desc = of.llama_graph(layers=2, tokens=MAX_ROWS, seq_len=128, hidden=1024, heads=16, kv_heads=4,
                          head_dim=64, inter=2048, dtype="bf16")
    g = of.build_graph(desc)
    sess = of.Session(g, of.partition(g, []), {"lanes": 3})
    host = llama_inputs(desc, MAX_ROWS, seed=11)
    full, outs = {}, {}
    for name, arr in host.items():
        t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
        if g.description["tensors"][g.tensor_id(name)].get("dtype") == "bf16":
            t = t.to(torch.bfloat16)
        full[name] = t.contiguous()
    for t in g.description["tensors"]:
        if t["role"] == "output":
            outs[t["name"]] = torch.empty([MAX_ROWS] + list(t["shape"][1:]), dtype=torch.bfloat16, device="cuda")

    def bind_rows(r):
        for name, t in full.items():
            batched = g.description["tensors"][g.tensor_id(name)].get("batch", "batched") == "batched"
            sess.bind(name, t[:r] if batched else t)
        for name, t in outs.items():
            sess.bind(name, t[:r])
        return sess

    return desc, host, sess, outs, bind_rows


def test_calibrated_table_drives_the_engine(cuda):
    import torch
    desc, host, sess, outs, bind_rows = _setup()
    sel = sl.calibrate(bind_rows, [SEQ, SPLIT], [256, 512, 1024], reps=3, rounds=2)
    rep = sel.report()
    for line in rep["lines_ms"]:
        assert line["alpha_ms"] >= 0 and line["beta_ms_per_row"] > 0
        assert len(line["samples"]) == 3
    spec = sel.spec()
    assert spec["table"][0]["min_rows"] == 0
    for r in (384, 768, 1024):
        s = bind_rows(r)
        s.run(spec)
        torch.cuda.synchronize()
        got = {k: v[:r].float().cpu().numpy() for k, v in outs.items()}
        chosen = s.stats()["auto"]
        assert any(a["key"].endswith(f"|rows={r}") for a in chosen)
        # the table's pick, run directly, gives bit-identical outputs (same plan)
        s.run(sel.choose(r))
        torch.cuda.synchronize()
        for k, v in outs.items():
            assert np.array_equal(v[:r].float().cpu().numpy(), got[k]), (r, k)
        batched = {t["name"] for t in of.build_graph(desc).description["tensors"]
                   if t.get("batch", "batched") == "batched"}
        sub = {k: (v[:r] if k in batched else v) for k, v in host.items()}
        want = oracle.evaluate(desc, r, sub, exact=False)
        for k in want:
            assert rel_err(got[k], want[k]) < 2e-2, (r, k)


def test_op_costs_fit_from_trace(cuda):
    _, _, sess, _, bind_rows = _setup()
    pts = {r: sl.trace_op_times(bind_rows(r)) for r in (256, 1024)}
    costs = sl.fit_op_costs(pts)
    assert any(k.startswith("layer0.") for k in costs), sorted(costs)
    for op, (a, b) in costs.items():
        assert a >= 0 and b >= 0, op
    # 4x the rows costs more in total (single tiny ops can be launch-bound and noisy)
    assert sum(b for a, b in costs.values()) > 0
    assert sum(pts[1024].values()) > sum(pts[256].values())
