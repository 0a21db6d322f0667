"""Tensor-parallel host logic on CPU with a real world-size-2 gloo group:
per-rank llama_graph(tp=2) + shard_llama_weights, evaluated by the oracle with
the AllReduce replaced by torch.distributed.all_reduce, must equal the
unsharded tp=1 graph ("compare the TP=W output against the oracle's
unsharded graph")."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPE = dict(layers=2, tokens=64, seq_len=32, hidden=128, heads=4, kv_heads=2, head_dim=32,
             inter=256, dtype="f32")


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_2605_21603_b200 import opflow as of
    from paper_2605_21603_b200.workloads import llama_inputs, shard_llama_weights
    full_desc = of.llama_graph(tp=1, **SHAPE)
    full = llama_inputs(full_desc, SHAPE["tokens"], seed=5)
    shard_desc = of.llama_graph(tp=world, **SHAPE)
    shard = shard_llama_weights(full, rank, world, SHAPE["heads"], SHAPE["kv_heads"],
                                SHAPE["head_dim"], SHAPE["inter"])
    # every per-rank tensor shape must match the tp graph's declarations
    g = of.build_graph(shard_desc)
    for name, arr in shard.items():
        decl = g.tensors[g.tensor_id(name)].shape
        if g.description["tensors"][g.tensor_id(name)].get("batch", "batched") == "replicated":
            assert list(arr.shape) == decl, name

    def allreduce(x, ws):
        assert ws == world
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
        dist.all_reduce(t)
        return t.numpy()

    got = oracle.evaluate(shard_desc, SHAPE["tokens"], shard, exact=False, allreduce=allreduce)
    want = oracle.evaluate(full_desc, SHAPE["tokens"], full, exact=False)
    errs = {k: float(np.linalg.norm(got[k] - want[k]) / np.linalg.norm(want[k])) for k in want}
    q.put((rank, errs))
    dist.destroy_process_group()


def test_tp2_sharding_equals_unsharded_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, errs in res:
        for k, e in errs.items():
            assert e < 1e-5, (rank, k, e)
