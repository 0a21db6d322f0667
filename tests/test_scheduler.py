"""Host-side scheduling contract + Algorithm 1 (no GPU): the SPEC's acceptance
properties for sched_api / dataflow_mem / engine, checked on
the device-free planner (opf_dry_run: the same code that plans GPU runs)."""
import json
import random

import pytest

from paper_2605_21603_b200 import opflow as of
from util import random_graph, unit_costs

pytestmark = pytest.mark.usefixtures("built")
R = of.PartitionRule


def plan_of(desc, rules=()):
    g = of.build_graph(desc)
    return g, of.partition(g, list(rules))


class Greedy(of.Scheduler):
    """'while unfinished: execute every ready op' (SPEC liveness property)."""

    def __init__(self, sizes, lanes=3, seed=0):
        self.sizes, self.lanes = sizes, lanes
        self.rng = random.Random(seed)
        self.cache_key = f"greedy{sizes}{seed}"

    def schedule(self, ctx):
        ctx.split(self.sizes)
        while ctx.unfinished():
            for u in range(len(self.sizes)):
                for h in ctx.get_ready_ops(u):
                    ctx.execute(h, lane=self.rng.randrange(self.lanes))


def random_sizes(rng, rows):
    n = rng.randint(1, min(4, rows))
    cuts = sorted(rng.sample(range(1, rows), n - 1)) if n > 1 else []
    return [b - a for a, b in zip([0] + cuts, cuts + [rows])]


def test_deadlock_freedom_1000_instances():
    rng = random.Random(7)
    for trial in range(1000):
        desc = random_graph(rng, min_ops=2, max_ops=16, batch=8)
        g, p = plan_of(desc, [R.by_func("All*")] if trial % 2 else [])
        sched, stats = of.dry_run(g, p, Greedy(random_sizes(rng, 8), seed=trial), rows=8)
        n_sg = p.size()
        covered = sum((d["u1"] - d["u0"]) * len(d["subgraphs"]) for d in sched["dispatches"])
        assert covered == n_sg * len({u for d in sched["dispatches"] for u in range(d["u0"], d["u1"])})
        assert stats["last"]["copied_elements"] == 0
        assert stats["last"]["end_live_tensors"] == 0


def test_sequential_single_lane_and_order():
    g, p = plan_of(of.dense_tp_graph(2, 8, 4, costs=unit_costs()), [R.by_func("AllReduce")])
    sched, stats = of.dry_run(g, p, {"name": "sequential"})
    assert [d["subgraphs"] for d in sched["dispatches"]] == [[i] for i in range(p.size())]
    assert {d["lane"] for d in sched["dispatches"]} == {0}
    assert all(d["wait_on"] == [] for d in sched["dispatches"])
    assert stats["last"]["lanes_used"] == 1


def test_split_sizes_and_zero_copy_views():
    g, p = plan_of(of.dense_tp_graph(1, 1024, 512, dtype="f32", costs=unit_costs()), [R.by_func("AllReduce")])
    sched, stats = of.dry_run(g, p, {"name": "split_overlap", "sizes": [512, 512]})
    # split [512,512] of [1024,512] -> element offsets 0 and 262144
    firsts = [d for d in sched["dispatches"] if d["subgraphs"] == [0]]
    offs = sorted(d["launches"][0]["in"][0]["elem_offset"] for d in firsts)
    assert offs == [0, 262144]
    assert all(d["rows"] == 512 for d in sched["dispatches"])
    assert stats["last"]["copied_elements"] == 0


def test_merge_uses_merge_buffer_and_fallback_copies():
    desc = of.moe_ep_graph(2, 8, 4, costs=unit_costs())
    rules = [R.by_module("layer*.attn"), R.by_module("layer*.moe.dispatch"),
             R.by_module("layer*.moe.experts"), R.by_module("layer*.moe.combine")]
    g, p = plan_of(desc, rules)
    sched, stats = of.dry_run(g, p, {"name": "dbo"})
    merged = [d for d in sched["dispatches"] if d["kind"] == "merged"]
    assert [d["labels"][0] for d in merged] == ["layer0.attn", "layer1.attn"]
    assert all(d["rows"] == 8 for d in merged)
    assert stats["last"]["copied_elements"] == 0
    # layer1.attn reads filler#4 outputs of both halves as ONE contiguous view
    m1 = merged[1]["launches"][0]["in"][0]
    assert m1["shape"][0] == 8
    _, stats_fb = of.dry_run(g, p, {"name": "dbo"}, config={"prealloc": False})
    assert stats_fb["last"]["copied_elements"] > 0


def test_dbo_interleaves_comm_and_compute_lanes():
    g, p = plan_of(of.moe_ep_graph(2, 8, 4, costs=unit_costs()),
                   [R.by_module("layer*.attn"), R.by_module("layer*.moe.dispatch"),
                    R.by_module("layer*.moe.experts"), R.by_module("layer*.moe.combine")])
    sched, _ = of.dry_run(g, p, {"name": "dbo"})
    lanes = {d["labels"][0].split(".")[-1]: d["lane"] for d in sched["dispatches"]}
    assert lanes["dispatch"] == 2 and lanes["combine"] == 2 and lanes["experts"] == 0
    assert any(d["wait_on"] for d in sched["dispatches"])  # cross-lane events


def test_fuse_norm_comm_replacement():
    g, p = plan_of(of.fuse_chain_graph(2, 8, 4, costs=unit_costs()),
                   [R.by_func("AllReduce"), R.by_func("RowScale")])
    sched, stats = of.dry_run(g, p, {"name": "fuse_norm_comm"})
    fused = [d for d in sched["dispatches"] if d["kind"] == "fused"]
    assert len(fused) == 4 and all(d["replace_fn"] == "allreduce_rowscale" for d in fused)
    assert all(d["lane"] == 2 for d in fused)
    assert stats["last"]["end_live_tensors"] == 0
    with pytest.raises(of.Error) as e:
        of.dry_run(*plan_of(of.fuse_chain_graph(2, 8, 4, costs=unit_costs()), []), {"name": "fuse_norm_comm"})
    assert e.value.code == of.Errc.MissingPattern
    with pytest.raises(of.Error) as e:
        of.dry_run(*plan_of(of.dense_tp_graph(2, 8, 4, costs=unit_costs()), []), {"name": "dbo"})
    assert e.value.code == of.Errc.MissingLabels


def test_plan_cache_hit_second_forward():
    g, p = plan_of(of.dense_tp_graph(2, 8, 4, costs=unit_costs()), [R.by_func("AllReduce")])
    _, stats = of.dry_run(g, p, {"name": "split_overlap"}, repeats=3)
    assert stats["plan_cache_misses"] == 1 and stats["plan_cache_hits"] == 2


def test_threshold_guard_falls_back_to_sequential():
    g, p = plan_of(of.dense_tp_graph(2, 8, 4, costs=unit_costs()), [R.by_func("AllReduce")])
    s1, _ = of.dry_run(g, p, {"name": "split_overlap", "threshold": 100})
    s0, _ = of.dry_run(g, p, {"name": "sequential"})
    assert [(d["subgraphs"], d["lane"], d["rows"]) for d in s1["dispatches"]] == \
           [(d["subgraphs"], d["lane"], d["rows"]) for d in s0["dispatches"]]


class Scripted(of.Scheduler):
    def __init__(self, fn, key):
        self.fn, self.cache_key = fn, key

    def schedule(self, ctx):
        self.fn(ctx)


@pytest.mark.parametrize("case,code", [
    ("split_twice", "AlreadySplit"), ("bad_sizes", "SizeMismatch"), ("not_ready", "NotReady"),
    ("dup", "DuplicateHandle"), ("incomplete", "IncompleteSchedule"),
    ("merge_gap", "MergeAcrossSplits"), ("bad_ubatch", "InvalidUbatch"),
    ("bad_replace", "SignatureMismatch"),
])
def test_sched_api_errors(case, code):
    g, p = plan_of(of.dense_tp_graph(1, 8, 4, costs=unit_costs()), [R.by_func("AllReduce")])

    def fn(ctx):
        if case == "split_twice":
            ctx.split([4, 4]); ctx.split([8])
        elif case == "bad_sizes":
            ctx.split([4, 5])
        elif case == "not_ready":
            ctx.execute(ctx.handle(1, 0))
        elif case == "dup":
            h = ctx.handle(0, 0); ctx.execute([h, h])
        elif case == "incomplete":
            ctx.execute(ctx.handle(0, 0))
        elif case == "merge_gap":
            ctx.split([2, 2, 4]); ctx.execute([ctx.handle(0, 0), ctx.handle(0, 2)])
        elif case == "bad_ubatch":
            ctx.get_ready_ops(3)
        elif case == "bad_replace":
            ctx.split([8]); ctx.execute(ctx.handle(0, 0)); ctx.execute([ctx.handle(1, 0), ctx.handle(2, 0)], 0, "nope")
    with pytest.raises(of.Error) as e:
        of.dry_run(g, p, Scripted(fn, case), rows=8)
    assert e.value.code == getattr(of.Errc, code)


def test_ready_frontier_matches_bruteforce():
    rng = random.Random(11)
    for trial in range(100):
        g, p = plan_of(random_graph(rng, batch=4), [R.by_func("*")] if trial % 3 == 0 else [R.by_module("m1")])
        seen = []

        def fn(ctx):
            done = set()
            while ctx.unfinished():
                ready = [h.subgraph for h in ctx.get_ready_ops(0)]
                want = [s for s in range(p.size()) if s not in done and all(q in done for q in p.sg_pred[s])]
                assert ready == want
                pick = rng.choice(ready)
                ctx.execute(ctx.handle(pick, 0))
                done.add(pick)
                seen.append(pick)
        of.dry_run(g, p, Scripted(fn, f"bf{trial}"), rows=4)
        assert sorted(seen) == list(range(p.size()))


def test_refcount_gc_reuses_arena():
    # chain graph: with GC the peak live bytes stay far below the sum of all
    # intermediates (SPEC: peak with GC <= peak without)
    g, p = plan_of(of.dense_tp_graph(8, 64, 64, dtype="f32", costs=unit_costs()),
                   [R.by_module("layer*")])
    _, stats = of.dry_run(g, p, {"name": "sequential"})
    per_tensor = 64 * 64 * 4
    assert stats["last"]["peak_live_bytes"] <= 6 * per_tensor  # independent of depth (8 layers)
    assert stats["last"]["plan_arena_bytes"] <= 8 * per_tensor


def test_llama_schedules_plan():
    desc = of.llama_graph(layers=2, tokens=1024, seq_len=256, hidden=256, heads=8, kv_heads=2,
                          head_dim=32, inter=512, tp=2, dtype="bf16")
    g, p = plan_of(desc, [R.by_func("AllReduce"), R.by_func("add_rmsnorm")])
    for strat in [{"name": "sequential"}, {"name": "split_overlap", "align": 256},
                  {"name": "fuse_norm_comm", "align": 256},
                  {"name": "split_overlap", "align": 256, "lane_mode": "ubatch", "n_microbatches": 4}]:
        sched, stats = of.dry_run(g, p, strat)
        assert stats["last"]["copied_elements"] == 0 and stats["last"]["end_live_tensors"] == 0
        for d in sched["dispatches"]:
            assert d["rows"] % 256 == 0
    sched, _ = of.dry_run(g, p, {"name": "fuse_norm_comm", "align": 256})
    fused = [d for d in sched["dispatches"] if d["kind"] == "fused"]
    assert fused and {d["replace_fn"] for d in fused} == {"allreduce_add_rmsnorm"}


def test_schedules_are_race_free():
    """Static race detection over compiled schedules (random graphs, random
    splits / merges / lanes): no two unordered dispatches touch overlapping
    arena bytes with a write."""
    from paper_2605_21603_b200.racecheck import find_races
    rng = random.Random(2024)

    class RandomStrategy(of.Scheduler):
        def __init__(self, seed):
            self.rng = random.Random(seed)
            self.cache_key = f"rs{seed}"

        def schedule(self, ctx):
            sizes = random_sizes(self.rng, ctx.rows)
            ctx.split(sizes)
            n_u = len(sizes)
            while ctx.unfinished():
                ready = {u: ctx.get_ready_ops(u) for u in range(n_u)}
                for u in range(n_u):
                    if not ready[u]:
                        continue
                    h = self.rng.choice(ready[u])
                    group, v = [h], u + 1
                    while v < n_u and self.rng.random() < 0.5 and any(x.subgraph == h.subgraph for x in ready[v]):
                        group.append(ctx.handle(h.subgraph, v))
                        v += 1
                    ctx.execute(group, lane=self.rng.randrange(3))
                    break

    for trial in range(300):
        desc = random_graph(rng, batch=12, hidden=16)
        g, p = plan_of(desc, [R.by_func("All*")] if trial % 2 else [R.by_module("m0")])
        for cfg in ({}, {"prealloc": False}):
            sched, stats = of.dry_run(g, p, RandomStrategy(trial), rows=12, config=cfg)
            races = find_races(sched)
            assert not races, (trial, cfg, races[:3])
    # the Llama schedules the bench runs
    desc = of.llama_graph(layers=2, tokens=1024, seq_len=256, hidden=256, heads=8, kv_heads=2,
                          head_dim=32, inter=512, tp=2, dtype="bf16")
    g, p = plan_of(desc, [R.by_func("AllReduce"), R.by_func("add_rmsnorm")])
    for strat in [{"name": "split_overlap", "align": 256, "lane_mode": "ubatch"},
                  {"name": "fuse_norm_comm", "align": 256}, {"name": "split_overlap", "align": 256}]:
        sched, _ = of.dry_run(g, p, strat)
        assert not find_races(sched)


def test_fuse_gemm_folds_row_parallel_matmul_into_the_allreduce():
    """fuse_norm_comm + fuse_gemm: an isolated o_proj / down MatMul subgraph joins
    its (AllReduce, add_rmsnorm) pair as ONE matmul_allreduce_add_rmsnorm
    dispatch (inputs a, w, x, g -> outputs x1, h) on the network lane; without
    the isolating rules the plan keeps the plain pairs."""
    desc = of.llama_graph(layers=2, tokens=512, seq_len=128, hidden=1024, heads=16, kv_heads=4, head_dim=64,
                          inter=2048, tp=2, dtype="bf16")
    g = of.build_graph(desc)
    rules = [R.by_module("layer*.attn.o"), R.by_module("layer*.mlp.down"), R.by_func("AllReduce"),
             R.by_func("add_rmsnorm")]
    p = of.partition(g, rules)
    sched, _ = of.dry_run(g, p, {"name": "fuse_norm_comm", "fuse_gemm": 1, "threshold": 1 << 20})
    fused = [d for d in sched["dispatches"] if d["replace_fn"] == "matmul_allreduce_add_rmsnorm"]
    assert [[g.ops[o].name for s in d["subgraphs"] for o in p.subgraphs[s].ops] for d in fused] == [
        ["layer0.o_proj", "layer0.o_allreduce", "layer0.attn_resid_norm"],
        ["layer0.down", "layer0.down_allreduce", "layer0.mlp_resid_norm"],
        ["layer1.o_proj", "layer1.o_allreduce", "layer1.attn_resid_norm"]]
    for d in fused:
        (l,) = d["launches"]
        names = [g.tensors[v["tensor"]].name for v in l["in"]]
        assert names[1].endswith((".o.w", ".down.w")) and names[3].endswith("norm.w"), names
        assert l["prepacked"] == l["in"][1]["tensor"]  # packed once per binding: K-major tcgen05 B operand
        assert len(l["out"]) == 2 and d["lane"] == 2
    # the last layer's down feeds an ElemAdd: plain AllReduce stays
    assert any(d["replace_fn"] == "" and [g.ops[o].name for s in d["subgraphs"] for o in p.subgraphs[s].ops]
               == ["layer1.down_allreduce"] for d in sched["dispatches"])
    # without isolating rules the MatMuls sit inside fillers: pairs only
    p2 = of.partition(g, [R.by_func("AllReduce"), R.by_func("add_rmsnorm")])
    s2, _ = of.dry_run(g, p2, {"name": "fuse_norm_comm", "fuse_gemm": 1})
    assert {d["replace_fn"] for d in s2["dispatches"]} == {"", "allreduce_add_rmsnorm"}


def test_residual_norm_epilogue_fusion_plan():
    """Peephole fusion plans MatMul -> add_rmsnorm as one epi-4 MatMul launch
    (inputs a, w, residual, gamma; outputs x1, h) when the residual is available
    at the MatMul's position; fuse_addnorm=false keeps them apart."""
    desc = of.llama_graph(layers=2, tokens=512, seq_len=128, hidden=512, heads=4, kv_heads=2, head_dim=128,
                          inter=1024, dtype="bf16")
    g = of.build_graph(desc)
    p = of.partition(g, [])
    sched, _ = of.dry_run(g, p, {"name": "sequential"})
    ls = [l for d in sched["dispatches"] for l in d["launches"]]
    fused = [l for l in ls if "resid_norm" in l["name"] and "+" in l["name"]]
    assert [l["name"] for l in fused] == ["layer0.o_proj+layer0.attn_resid_norm",
                                          "layer0.down+layer0.mlp_resid_norm",
                                          "layer1.o_proj+layer1.attn_resid_norm"]
    for l in fused:
        assert len(l["in"]) == 4 and len(l["out"]) == 2 and l["ws_bytes"] >= 512 * 2 * 4
    plain, _ = of.dry_run(g, p, {"name": "sequential"}, config={"fuse_addnorm": False})
    assert not any("resid_norm" in l["name"] and "+" in l["name"]
                   for d in plain["dispatches"] for l in d["launches"])


def test_fused_epilogue_keeps_arena_liveness():
    """An op run inside its producer's GEMM epilogue (add_rmsnorm) still retires
    its inputs at its own position: the 32-layer Llama-3-8B plan at 8192 rows
    stays under 1 GiB of arena with the fusion on."""
    desc = of.llama_graph(layers=32, tokens=8192, seq_len=1024, hidden=4096, heads=32, kv_heads=8,
                          head_dim=128, inter=14336, dtype="bf16")
    g = of.build_graph(desc)
    p = of.partition(g, [])
    _, fused = of.dry_run(g, p, {"name": "sequential"}, rows=8192)
    _, plain = of.dry_run(g, p, {"name": "sequential"}, rows=8192, config={"fuse_addnorm": False})
    assert fused["last"]["plan_arena_bytes"] < (1 << 30)
    assert fused["last"]["plan_arena_bytes"] < 2 * plain["last"]["plan_arena_bytes"]


def test_sequential_fallback_is_all_or_nothing():
    """execute([a, b]) without a replacement runs a then b in order (b may
    depend on a).  If a later handle is not ready, nothing is recorded: the
    context is unchanged (SPEC: scheduler-visible state is totally ordered
    and reproducible), so a strategy that catches NotReady sees no phantom
    dispatch of `a`."""
    g, p = plan_of(of.dense_tp_graph(1, 8, 4, costs=unit_costs()), [R.by_func("AllReduce")])
    seen = {}

    def fn(ctx):
        ctx.split([8])
        with pytest.raises(of.Error) as e:
            ctx.execute([ctx.handle(0, 0), ctx.handle(2, 0)])  # 2 needs 1, which is not in the list
        assert e.value.code == of.Errc.NotReady
        seen["ready_after_failure"] = [h.subgraph for h in ctx.get_ready_ops(0)]
        ctx.execute([ctx.handle(0, 0), ctx.handle(1, 0), ctx.handle(2, 0)])  # chained: fine in order

    sched, _ = of.dry_run(g, p, Scripted(fn, "atomic"), rows=8)
    assert seen["ready_after_failure"] == [0]
    assert [d["subgraphs"] for d in sched["dispatches"]] == [[0], [1], [2]]
