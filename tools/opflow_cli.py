#!/usr/bin/env python3
"""Thin scenario driver for the B200 backend (SPEC.md:527-586 `cli`).

  opflow_cli.py validate --config scenario.json          (CPU: no GPU needed)
  opflow_cli.py run      --config scenario.json --out DIR [--strategy NAME] [--seed N]
  opflow_cli.py sweep    --config scenario.json --out DIR --axis rows --values 1024,2048,...

Scenario (JSON):
  {"graph": {"builder": "llama", "params": {...}}   |  {"description": {...GraphDescription...}},
   "rules": [{"kind": "func", "pattern": "AllReduce"}, ...],
   "strategy": {"name": "split_overlap", ...},
   "workload": [{"rows": 8192}], "seed": 2026, "config": {"lanes": 3}}

`validate` builds the graph, partitions it, plans the configured strategy on the
device-free planner and checks the invariants (plan validity, Algorithm-1
conservation: end live set = outputs, zero copies, static race freedom).
`run` executes sequential + the strategy on cuda:0 and writes metrics.json
(ms / tokens per second / speedup_vs_sequential / plan-cache hit rate /
copied elements / arena bytes) plus one Trace Event JSON per run
({name, cat, ph:"X", ts, dur, pid, tid = lane}).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_21603_b200 import opflow as of  # noqa: E402
from paper_2605_21603_b200.racecheck import find_races  # noqa: E402


def load(path):
    with open(path) as f:
        return json.load(f)


def description(sc, rows=None):
    g = sc["graph"]
    if "description" in g:
        return json.dumps(g["description"])
    params = dict(g.get("params", {}))
    if rows is not None:
        key = "tokens" if g["builder"] in ("llama", "llama_decode", "toy_decoder") else "batch"
        params[key] = rows
    return of.builder_json(g["builder"], **params)


def rules(sc):
    return [of.PartitionRule(r["kind"], r["pattern"]) for r in sc.get("rules", [])]


def cmd_validate(sc, args):
    desc = description(sc)
    g = of.build_graph(desc)
    plan = of.partition(g, rules(sc))
    of.validate_plan(plan, g)
    report = {"ops": len(g.ops), "subgraphs": plan.size(), "labels": [s.label for s in plan.subgraphs]}
    for w in sc.get("workload", [{"rows": None}]):
        sched, stats = of.dry_run(g, plan, sc.get("strategy", {"name": "sequential"}), rows=w.get("rows"),
                                  config=sc.get("config"))
        last = stats["last"]
        races = find_races(sched)
        ok = last["copied_elements"] == 0 and last["end_live_tensors"] == 0 and not races
        report.setdefault("workloads", []).append(
            {"rows": w.get("rows"), "dispatches": last["dispatches"], "launches": last["launches"],
             "lanes_used": last["lanes_used"], "copied_elements": last["copied_elements"],
             "end_live_tensors": last["end_live_tensors"], "races": len(races), "ok": ok})
    print(json.dumps(report, indent=1))
    return 0 if all(w["ok"] for w in report["workloads"]) else 1


def _run_one(sc, strategy, rows, seed, steps=10, warmup=3):
    import numpy as np
    import torch
    from paper_2605_21603_b200.workloads import llama_inputs, standin_inputs
    desc = description(sc, rows)
    g = of.build_graph(desc)
    plan = of.partition(g, rules(sc))
    sess = of.Session(g, plan, sc.get("config", {"lanes": 3}))
    llama = any(t.get("dtype") == "bf16" or t["name"] == "positions" for t in json.loads(desc)["tensors"])
    host = (llama_inputs if llama else standin_inputs)(desc, rows, seed=seed)
    keep = {}
    for name, arr in host.items():
        t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
        if g.description["tensors"][g.tensor_id(name)].get("dtype") == "bf16":
            t = t.to(torch.bfloat16)
        keep[name] = t
        sess.bind(name, t)
    for t in g.description["tensors"]:
        if t["role"] == "output":
            shape = list(t["shape"])
            shape[0] = rows
            dt = {"i64": torch.int64, "f32": torch.float32, "bf16": torch.bfloat16}[t.get("dtype", "i64")]
            keep[t["name"]] = torch.empty(shape, dtype=dt, device="cuda")
            sess.bind(t["name"], keep[t["name"]])
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        sess.run(strategy, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(steps):
        sess.run(strategy, s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    st = sess.stats()
    trace = sess.trace()
    return ms, st, trace


def cmd_run(sc, args, rows_list=None):
    os.makedirs(args.out, exist_ok=True)
    strat = sc.get("strategy", {"name": "sequential"})
    if args.strategy:
        strat = dict(strat, name=args.strategy)
    seed = args.seed if args.seed is not None else sc.get("seed", 0)
    runs = []
    for w in (rows_list or sc.get("workload", [{"rows": 1024}])):
        rows = w["rows"]
        ms_seq, _, tr_seq = _run_one(sc, {"name": "sequential"}, rows, seed)
        ms, st, tr = _run_one(sc, strat, rows, seed)
        hits, miss = st["plan_cache_hits"], st["plan_cache_misses"]
        runs.append({"rows": rows, "strategy": strat, "ms_per_forward": ms,
                     "tokens_per_s": rows / (ms / 1e3), "sequential_ms": ms_seq,
                     "speedup_vs_sequential": ms_seq / ms,
                     "plan_cache_hit_rate": hits / max(1, hits + miss),
                     "total_copied_elements": st["last"]["copied_elements"],
                     "peak_live_bytes": st["last"]["peak_live_bytes"],
                     "end_live_tensors": st["last"]["end_live_tensors"],
                     "arena_bytes": st["arena_bytes"]})
        for name, t in (("sequential", tr_seq), (strat["name"], tr)):
            with open(os.path.join(args.out, f"trace_{name}_rows{rows}.json"), "w") as f:
                json.dump(t, f)
    with open(os.path.join(args.out, "metrics.json"), "w") as f:
        json.dump({"runs": runs}, f, indent=1)
    print(json.dumps({"runs": runs}))
    return 0


def cmd_sweep(sc, args):
    vals = [int(v) for v in args.values.split(",")]
    rc = cmd_run(sc, args, [{"rows": v} for v in vals])
    with open(os.path.join(args.out, "metrics.json")) as f:
        runs = json.load(f)["runs"]
    with open(os.path.join(args.out, "sweep.csv"), "w") as f:
        f.write("rows,ms_per_forward,sequential_ms,speedup_vs_sequential\n")
        for r in runs:
            f.write(f"{r['rows']},{r['ms_per_forward']:.4f},{r['sequential_ms']:.4f},"
                    f"{r['speedup_vs_sequential']:.4f}\n")
    return rc


def main(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("cmd", choices=["validate", "run", "sweep"])
    p.add_argument("--config", required=True)
    p.add_argument("--out", default="opflow_out")
    p.add_argument("--seed", type=int)
    p.add_argument("--strategy")
    p.add_argument("--axis", default="rows")
    p.add_argument("--values", default="")
    args = p.parse_args(argv)
    sc = load(args.config)
    try:
        return {"validate": cmd_validate, "run": cmd_run, "sweep": cmd_sweep}[args.cmd](sc, args)
    except of.Error as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
