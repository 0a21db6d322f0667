"""One rank of a real multi-process peer-memory run (tests/test_gpu_multiproc.py).

Launched W times as separate processes.  Every rank is its own CUDA context
(all W on cuda:0 under `gpurun`, one per GPU on a multi-GPU box), owns a
peer-only communicator (`Comm.peer`: no NCCL, which refuses two ranks on one
device) and exchanges real CUDA-IPC handles for its window and its symmetric
session arena over a gloo process group.  So the cross-process parts of the
protocol run for real: IPC mapping, `st.release.sys` / `ld.acquire.sys`
flag barriers between contexts, device epochs advancing across replays, and
the engine's window-error check.

Each case compares this rank's outputs with the unsharded oracle and prints
one JSON line {"rank", "case", "errors": {...}, "push_calls", ...}.

    python tests/mp_worker.py --rank R --world W --case ar|tp|tp_fuse|ep|timeout
(MASTER_ADDR / MASTER_PORT in the environment.)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

TP_SHAPE = dict(layers=2, tokens=256, seq_len=128, hidden=512, heads=8, kv_heads=4, head_dim=128, inter=1024)
EP_SHAPE = dict(layers=2, tokens=256, seq_len=128, hidden=256, heads=4, kv_heads=2, head_dim=128,
                experts=16, topk=4, moe_inter=128)


def _bind_all(torch, of, sess, g, arrays, outs):
    keep = {}
    for t in g.description["tensors"]:
        name = t["name"]
        if t["role"] == "output":
            keep[name] = torch.empty(list(t["shape"]), dtype=torch.bfloat16, device="cuda")
            outs[name] = keep[name]
        elif t["role"] in ("input", "weight"):
            x = torch.from_numpy(np.ascontiguousarray(arrays[name])).cuda()
            if t.get("dtype") == "bf16":
                x = x.to(torch.bfloat16)
            keep[name] = x
        else:
            continue
        sess.bind(name, keep[name])
    return keep


def case_ar(torch, of, comm, rank, world, res):
    """allreduce_add_rmsnorm in every form (pull, two-shot, push, auto) and the
    AllReduce kind, rows divisible and not divisible by the world size."""
    from oracle import oracle
    from paper_2605_21603_b200.workloads import rel_err
    H = 4096
    tb = lambda a: torch.from_numpy(a.astype(np.float32)).cuda().to(torch.bfloat16)
    stream = torch.cuda.Stream()
    for mode, name in ((1, "pull"), (2, "twoshot"), (3, "push"), (0, "auto")):
        for rows in (64, 61):
            rng = np.random.default_rng(1000 + rows)  # same global data on every rank
            x = tb(rng.uniform(-1, 1, (rows, H)))
            g = tb(1 + 0.1 * rng.uniform(-1, 1, H))
            op = {"name": "f", "kind": "Custom", "inputs": [], "outputs": [],
                  "attrs": {"custom_name": "allreduce_add_rmsnorm", "world_size": world,
                            "params": {"eps": 1e-5, "ar_mode": mode}}}
            for it in range(3):  # device epochs advance across calls
                parts = [tb(rng.uniform(-1, 1, (rows, H))) for _ in range(world)]
                x1, y = torch.empty_like(x), torch.empty_like(x)
                torch.cuda.synchronize()
                of.launch(op, [parts[rank], x, g], [x1, y], rows, stream, comm=comm)
                torch.cuda.synchronize()
                s = x.float().cpu().numpy() + sum(p.float().cpu().numpy() for p in parts)
                want_h = oracle.rmsnorm(s, g.float().cpu().numpy(), 1e-5)
                key = f"{name}_r{rows}"
                res["errors"][key + "_x1"] = max(res["errors"].get(key + "_x1", 0.0),
                                                 rel_err(x1.float().cpu().numpy(), s))
                res["errors"][key + "_h"] = max(res["errors"].get(key + "_h", 0.0),
                                                rel_err(y.float().cpu().numpy(), want_h))
    # the AllReduce kind (one-shot peer all-reduce; a peer-only comm takes it at any size)
    for rows in (64, 1024):
        rng = np.random.default_rng(77 + rows)
        parts = [tb(rng.uniform(-1, 1, (rows, H))) for _ in range(world)]
        out = torch.empty_like(parts[0])
        ar = {"name": "ar", "kind": "AllReduce", "inputs": [], "outputs": [], "attrs": {"world_size": world}}
        of.launch(ar, [parts[rank]], [out], rows, stream, comm=comm)
        torch.cuda.synchronize()
        want = sum(p.float().cpu().numpy() for p in parts)
        res["errors"][f"allreduce_r{rows}"] = rel_err(out.float().cpu().numpy(), want)


def _tp_run(torch, of, comm, rank, world, strategies, rules, shape, res):
    from oracle import oracle
    from paper_2605_21603_b200.workloads import llama_inputs, rel_err, shard_llama_weights
    T = shape["tokens"]
    full_desc = of.llama_graph(tp=1, dtype="bf16", **shape)
    full = llama_inputs(full_desc, T, seed=9)
    want = oracle.evaluate(full_desc, T, full, exact=False)
    desc = of.llama_graph(tp=world, dtype="bf16", **shape)
    shard = shard_llama_weights(full, rank, world, shape["heads"], shape["kv_heads"], shape["head_dim"],
                                shape["inter"])
    g = of.build_graph(desc)
    sess = of.Session(g, of.partition(g, rules), {"lanes": 3}, comm)
    outs = {}
    keep = _bind_all(torch, of, sess, g, shard, outs)  # noqa: F841
    stream = torch.cuda.Stream()
    for key, spec in strategies.items():
        for o in outs.values():
            o.fill_(float("nan"))
        for _ in range(3):  # replays: epochs advance on the device
            sess.run(spec, stream)
        sess.check()  # raises SchedulerError if a barrier timed out
        torch.cuda.synchronize()
        for name, t in outs.items():
            res["errors"][f"{key}:{name}"] = rel_err(t.float().cpu().numpy(), want[name])
        # replicated activations: every rank must hold identical bytes
        res.setdefault("digest", {})[key] = {n: float(t.float().sum().item()) for n, t in outs.items()}
    res["stats"] = sess.stats()["last"]


def case_tp(torch, of, comm, rank, world, res):
    R = of.PartitionRule
    strategies = {"sequential": {"name": "sequential"},
                  "nanoflow": {"name": "split_overlap", "n_microbatches": 2, "align": 128},
                  "tokenweave": {"name": "fuse_norm_comm", "align": 128}}
    _tp_run(torch, of, comm, rank, world, strategies, [R.by_func("AllReduce"), R.by_func("add_rmsnorm")],
            TP_SHAPE, res)


def case_tp_fuse(torch, of, comm, rank, world, res):
    """Row-parallel GEMM whose epilogue pushes partial slabs into the owner
    rank's window (another process's memory) + reduce + add + RMSNorm."""
    R = of.PartitionRule
    rules = [R.by_module("layer*.attn.o"), R.by_module("layer*.mlp.down"), R.by_func("AllReduce"),
             R.by_func("add_rmsnorm")]
    shape = dict(TP_SHAPE, tokens=512, kv_heads=max(TP_SHAPE["kv_heads"], world))
    strategies = {"gemm_push": {"name": "fuse_norm_comm", "fuse_gemm": 1, "threshold": 1 << 20},
                  "gemm_push_split": {"name": "fuse_norm_comm", "fuse_gemm": 1, "align": 128}}
    _tp_run(torch, of, comm, rank, world, strategies, rules, shape, res)
    res["push_calls"] = comm.push_calls()


def case_ep(torch, of, comm, rank, world, res):
    """Expert-parallel Qwen3-MoE layers: dispatch writes rows straight into the
    owner process's arena, combine writes results back (CUDA IPC)."""
    from oracle import oracle
    from paper_2605_21603_b200.workloads import llama_inputs, rel_err
    R = of.PartitionRule
    T, E = EP_SHAPE["tokens"], EP_SHAPE["experts"]
    El = E // world
    full = of.qwen3_moe_graph(**EP_SHAPE)
    host = llama_inputs(full, T, seed=5)
    rng = np.random.default_rng(world)
    xs = [np.ascontiguousarray(host["x"] + rng.uniform(-0.5, 0.5, host["x"].shape).astype(np.float32) * r)
          for r in range(world)]
    mine = dict(host, x=xs[rank])
    want = oracle.evaluate(full, T, mine, exact=False)
    arrays = {}
    for name, arr in mine.items():
        if name.startswith("layer") and ".experts." in name:
            arr = arr[rank * El:(rank + 1) * El]
        arrays[name] = arr
    desc = of.qwen3_moe_graph(**EP_SHAPE, ep=world)
    g = of.build_graph(desc)
    plan = of.partition(g, [R.by_module("layer*.attn"), R.by_module("layer*.moe.dispatch"),
                            R.by_module("layer*.moe.experts"), R.by_module("layer*.moe.combine")])
    sess = of.Session(g, plan, {"lanes": 3}, comm)
    outs = {}
    keep = _bind_all(torch, of, sess, g, arrays, outs)  # noqa: F841
    strategies = {"sequential": {"name": "sequential"}, "dbo": {"name": "dbo", "align": 128}}
    need = max(of.dry_run(g, plan, s, rows=T, config={"lanes": 3, "world": world})[1]["last"]["plan_arena_bytes"]
               for s in strategies.values())
    sess.enable_peer_arena(need)
    stream = torch.cuda.Stream()
    for key, spec in strategies.items():
        for o in outs.values():
            o.fill_(float("nan"))
        for _ in range(2):
            sess.run(spec, stream)
        sess.check()
        torch.cuda.synchronize()
        for name, t in outs.items():
            res["errors"][f"{key}:{name}"] = rel_err(t.float().cpu().numpy(), want[name])
    res["copied_elements"] = sess.stats()["last"]["copied_elements"]


def case_timeout(torch, of, comm, rank, world, res):
    """Rank 0 runs a collective its peer never joins: the barrier must time
    out, raise the window's error flag, and Session.check() must raise
    SchedulerError (not return wrong activations with status OK)."""
    import torch.distributed as dist
    if rank == 0:
        R = of.PartitionRule
        desc = of.llama_graph(tp=world, dtype="bf16", **TP_SHAPE)
        from paper_2605_21603_b200.workloads import llama_inputs
        arrays = llama_inputs(desc, TP_SHAPE["tokens"], seed=3)
        g = of.build_graph(desc)
        sess = of.Session(g, of.partition(g, [R.by_func("AllReduce")]), {"lanes": 1}, comm)
        outs = {}
        keep = _bind_all(torch, of, sess, g, arrays, outs)  # noqa: F841
        sess.run({"name": "sequential"}, torch.cuda.Stream())
        try:
            sess.check()
            res["raised"] = None
        except of.Error as e:
            res["raised"] = e.code.name
        res["window_error"] = comm.window_error()
    dist.barrier()


CASES = {"ar": case_ar, "tp": case_tp, "tp_fuse": case_tp_fuse, "ep": case_ep, "timeout": case_timeout}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--case", required=True, choices=sorted(CASES))
    ap.add_argument("--device", type=int, default=-1, help="-1: all ranks on cuda:0")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2605_21603_b200 import opflow as of
    dev = 0 if a.device < 0 else a.device
    torch.cuda.set_device(dev)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo", rank=a.rank, world_size=a.world)
    comm = of.Comm.peer(a.world, a.rank, dev)
    comm.enable_window(4 * 1024 * 4096 * 2)  # holds W=2..4 push planes of the 1024-row all-reduce
    res = {"rank": a.rank, "case": a.case, "errors": {}}
    CASES[a.case](torch, of, comm, a.rank, a.world, res)
    torch.cuda.synchronize()
    res["window_error"] = res.get("window_error", comm.window_error())
    dist.barrier()
    print("RESULT " + json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
