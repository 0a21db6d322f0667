"""GPU: tensor-parallel Llama layers (BASELINE configs[1..2]'s TP=W path) with
W virtual ranks sharing one B200.  Every rank binds its Megatron shard of the
full weights (shard_llama_weights) into llama_graph(tp=W); the AllReduce ops
run the peer-memory one-shot all-reduce over the ranks' windows, and the
TokenWeave strategy replaces AllReduce + add_rmsnorm by the fused peer-memory
kernel.  Each rank's output must equal the unsharded tp=1 oracle."""
import numpy as np
import pytest

from oracle import oracle
from paper_2605_21603_b200 import opflow as of
from paper_2605_21603_b200.workloads import llama_inputs, rel_err, shard_llama_weights

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("built")]
SHAPE = dict(layers=2, tokens=256, seq_len=128, hidden=512, heads=8, kv_heads=4, head_dim=128, inter=1024)
R = of.PartitionRule


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("strategy", [{"name": "sequential"},
                                      {"name": "split_overlap", "n_microbatches": 2, "align": 128},
                                      {"name": "fuse_norm_comm", "align": 128}])
def test_tp_llama_virtual_ranks_vs_unsharded_oracle(cuda, world, strategy):
    import torch
    T = SHAPE["tokens"]
    full_desc = of.llama_graph(tp=1, dtype="bf16", **SHAPE)
    full = llama_inputs(full_desc, T, seed=9)
    want = oracle.evaluate(full_desc, T, full, exact=False)
    desc = of.llama_graph(tp=world, dtype="bf16", **SHAPE)
    comms = of.Comm.virtual(world, 0, T * SHAPE["hidden"] * 2)
    # every kernel of every rank capped at 16 CTAs: all W ranks' cross-rank
    # barriers stay co-resident on the one GPU
    cfg = {"lanes": 3, "lane_sm_budget": [16, 16, 16]}
    sessions, keep, outs = [], [], []
    for r in range(world):
        shard = shard_llama_weights(full, r, world, SHAPE["heads"], SHAPE["kv_heads"], SHAPE["head_dim"],
                                    SHAPE["inter"])
        g = of.build_graph(desc)
        sess = of.Session(g, of.partition(g, [R.by_func("AllReduce"), R.by_func("add_rmsnorm")]), cfg, comms[r])
        k = {}
        for t in g.description["tensors"]:
            name = t["name"]
            if t["role"] == "output":
                k[name] = torch.empty(list(t["shape"]), dtype=torch.bfloat16, device="cuda")
                outs.append((r, name, k[name]))
            elif t["role"] in ("input", "weight"):
                x = torch.from_numpy(np.ascontiguousarray(shard[name])).cuda()
                if t.get("dtype") == "bf16":
                    x = x.to(torch.bfloat16)
                k[name] = x
            else:
                continue
            sess.bind(name, k[name])
        sessions.append(sess)
        keep.append(k)
    streams = [torch.cuda.Stream() for _ in range(world)]
    torch.cuda.synchronize()
    for r in range(world):
        sessions[r].prepare(strategy, streams[r])
    torch.cuda.synchronize()
    for _ in range(2):  # replays: device epochs advance across calls
        for r in range(world):
            sessions[r].run(strategy, streams[r])
    torch.cuda.synchronize()
    for c in comms:
        assert c.window_error() == 0
    for r, name, t in outs:
        err = rel_err(t.float().cpu().numpy(), want[name])
        assert err < 2e-2, (r, name, err)


FUSE_RULES = [R.by_module("layer*.attn.o"), R.by_module("layer*.mlp.down"), R.by_func("AllReduce"),
              R.by_func("add_rmsnorm")]


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("strategy,pushes", [
    ({"name": "fuse_norm_comm", "fuse_gemm": 1, "threshold": 1 << 20}, 3),  # unsplit: o, down, o
    ({"name": "fuse_norm_comm", "fuse_gemm": 1, "align": 128}, 6),  # two 256-row nano-batches
    ({"name": "fuse_norm_comm", "fuse_gemm": 1, "sizes": [128] * 4}, 0)])  # <= 128 rows: GEMM + p2p AR fallback
def test_tp_gemm_push_allreduce_vs_unsharded_oracle(cuda, world, strategy, pushes):
    """Row-parallel GEMM -> all-reduce -> add + RMSNorm as ONE op: the GEMM
    epilogue pushes each 32-row slab of its partial into the owner rank's
    window (this rank's slot) and counts it; the reduce kernel sums the slots,
    normalises its block, publishes x1 and gathers the other owners' x1.  Each
    rank's output equals the unsharded oracle; the push protocol actually ran
    (call epochs), and replays stay in lock-step."""
    import torch
    shape = dict(SHAPE, tokens=512, kv_heads=max(SHAPE["kv_heads"], world))
    T = shape["tokens"]
    full_desc = of.llama_graph(tp=1, dtype="bf16", **shape)
    full = llama_inputs(full_desc, T, seed=13)
    want = oracle.evaluate(full_desc, T, full, exact=False)
    desc = of.llama_graph(tp=world, dtype="bf16", **shape)
    comms = of.Comm.virtual(world, 0, 3 * T * shape["hidden"] * 2)
    # all W ranks' GEMMs and spinning reduce kernels must be co-resident on one GPU
    b = 16 if world <= 4 else 8
    cfg = {"lanes": 3, "lane_sm_budget": [b, b, b]}
    sessions, keep, outs = [], [], []
    for r in range(world):
        shard = shard_llama_weights(full, r, world, shape["heads"], shape["kv_heads"], shape["head_dim"],
                                    shape["inter"])
        g = of.build_graph(desc)
        sess = of.Session(g, of.partition(g, FUSE_RULES), cfg, comms[r])
        k = {}
        for t in g.description["tensors"]:
            name = t["name"]
            if t["role"] == "output":
                k[name] = torch.empty(list(t["shape"]), dtype=torch.bfloat16, device="cuda")
                outs.append((r, name, k[name]))
            elif t["role"] in ("input", "weight"):
                x = torch.from_numpy(np.ascontiguousarray(shard[name])).cuda()
                if t.get("dtype") == "bf16":
                    x = x.to(torch.bfloat16)
                k[name] = x
            else:
                continue
            sess.bind(name, k[name])
        sessions.append(sess)
        keep.append(k)
    streams = [torch.cuda.Stream() for _ in range(world)]
    torch.cuda.synchronize()
    for r in range(world):
        sessions[r].prepare(strategy, streams[r])
    torch.cuda.synchronize()
    reps = 3
    for _ in range(reps):
        for r in range(world):
            sessions[r].run(strategy, streams[r])
    torch.cuda.synchronize()
    for c in comms:
        assert c.window_error() == 0
        assert c.push_calls() == pushes * reps
    for r, name, t in outs:
        err = rel_err(t.float().cpu().numpy(), want[name])
        assert err < 2e-2, (r, name, err)
    # every rank holds the same replicated activations
    for name in {n for _, n, _ in outs}:
        ts = [t for _, n, t in outs if n == name]
        for t in ts[1:]:
            assert torch.equal(t, ts[0]), name
