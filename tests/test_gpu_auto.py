"""GPU: context-aware strategy selection ("auto": candidates timed on the device,
winner cached per row count) keeps parity and is visible in the stats; the SPEC
cli `run` writes metrics.json and Trace Event JSON."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle
from paper_2605_21603_b200 import opflow as of
from paper_2605_21603_b200.workloads import llama_inputs, rel_err
from test_gpu_parity import run_graph

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("built")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_auto_strategy_selection(cuda):
    desc = of.llama_graph(layers=2, tokens=512, seq_len=128, hidden=512, heads=4, kv_heads=2,
                          head_dim=128, inter=1024, dtype="bf16")
    host = llama_inputs(desc, 512, seed=3)
    want = oracle.evaluate(desc, 512, host, exact=False)
    auto = {"name": "auto", "reps": 3, "candidates": [
        {"name": "sequential"},
        {"name": "split_overlap", "n_microbatches": 2, "align": 128, "lane_mode": "ubatch"},
        {"name": "split_overlap", "n_microbatches": 4, "align": 128}]}
    got, sess = run_graph(desc, 512, host, auto, repeat=3)
    st = sess.stats()
    assert len(st["auto"]) == 1 and len(st["auto"][0]["ms"]) == 3
    chosen = json.loads(st["auto"][0]["chosen"])
    assert chosen in auto["candidates"]
    for k in want:
        assert rel_err(got[k], want[k]) < 2e-2


def test_cli_run_writes_metrics_and_traces(cuda, tmp_path):
    out = tmp_path / "o"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "opflow_cli.py"), "run",
                        "--config", os.path.join(ROOT, "scenarios", "dense_tp_split.json"),
                        "--out", str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    m = json.loads((out / "metrics.json").read_text())
    run = m["runs"][0]
    assert run["total_copied_elements"] == 0 and run["end_live_tensors"] == 0
    assert run["plan_cache_hit_rate"] > 0.5
    tr = json.loads((out / "trace_split_overlap_rows1024.json").read_text())
    assert tr and all(e["ph"] == "X" and {"name", "ts", "dur", "pid", "tid"} <= set(e) for e in tr)
    assert len({e["tid"] for e in tr}) >= 2  # more than one lane busy
