"""Test helpers: random graph generator modelled on the reference's
testutil::random_graph (/root/reference/proj/tests/test_util.hpp:42-106)."""
from __future__ import annotations

import json
import random

KINDS = ["MatMul", "ElemAdd", "RowScale", "AllReduce", "AllToAll", "Attention"]


def unit_costs():
    # /root/reference/proj/tests/test_partition.cpp:18-26
    return {"attention": [1.0, 0.1], "matmul": [1.0, 0.3], "allreduce": [1.0, 0.1],
            "alltoall": [1.0, 0.1], "rowscale": [1.0, 0.05]}


def random_graph(rng: random.Random, min_ops=4, max_ops=24, batch=8, hidden=4, dtype="i64",
                 region_tags=False) -> str:
    B, H = batch, hidden
    tensors = [{"name": "x", "shape": [B, H], "batch": "batched", "dtype": dtype, "role": "input"}]
    ops = []
    batched = ["x"]
    n = rng.randint(min_ops, max_ops)
    wc = 0
    for i in range(n):
        kind = rng.choice(KINDS)
        o = {"name": f"op{i}", "kind": kind, "module_path": f"m{i % 4}.op{i}", "outputs": [f"t{i}"],
             "attrs": {}}
        if kind == "MatMul":
            w = f"w{wc}"
            wc += 1
            tensors.append({"name": w, "shape": [H, H], "batch": "replicated", "dtype": dtype,
                            "role": "weight"})
            o["inputs"] = [rng.choice(batched), w]
        elif kind == "ElemAdd":
            o["inputs"] = [rng.choice(batched), rng.choice(batched)]
        elif kind == "AllReduce":
            o["inputs"] = [rng.choice(batched)]
            o["attrs"]["world_size"] = 2
        elif kind == "AllToAll":
            o["inputs"] = [rng.choice(batched)]
            o["attrs"]["seed"] = i + 17
        else:
            o["inputs"] = [rng.choice(batched)]
        o["cost"] = [rng.uniform(0.5, 4.0), rng.uniform(0.5, 4.0) / 8.0]
        if region_tags and rng.random() < 0.2:
            o["region_tags"] = ["hot"]
        tensors.append({"name": f"t{i}", "shape": [B, H], "batch": "batched", "dtype": dtype,
                        "role": "intermediate"})
        ops.append(o)
        batched.append(f"t{i}")
    consumed = {x for o in ops for x in o["inputs"]}
    for t in tensors:
        if t["role"] == "intermediate" and t["name"] not in consumed:
            t["role"] = "output"
    return json.dumps({"tensors": tensors, "operators": ops})


def shuffled(desc_json: str, rng: random.Random) -> str:
    d = json.loads(desc_json)
    rng.shuffle(d["operators"])
    return json.dumps(d)
