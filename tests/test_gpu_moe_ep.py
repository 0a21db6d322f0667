"""GPU: expert-parallel Qwen3-MoE layer over peer-memory all-to-all.

W virtual ranks share one B200 (the real multi-GPU path differs only in how
windows / arenas are mapped: CUDA IPC over NVLink instead of same-device
pointers).  Every rank has its own tokens and holds experts/W experts'
weights; dispatch writes rows straight into the owner's arena, combine writes
results straight back.  Each rank's output must equal the single-rank (ep=1)
oracle on its tokens with the full expert set."""
import numpy as np
import pytest

from oracle import oracle
from paper_2605_21603_b200 import opflow as of
from paper_2605_21603_b200.workloads import llama_inputs, rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("built")]
R = of.PartitionRule
SMALL = dict(layers=2, tokens=256, seq_len=128, hidden=256, heads=4, kv_heads=2, head_dim=128,
             experts=16, topk=4, moe_inter=128)
RULES = [R.by_module("layer*.attn"), R.by_module("layer*.moe.dispatch"),
         R.by_module("layer*.moe.experts"), R.by_module("layer*.moe.combine")]


def run_ep(world, strategy, repeats=2, skew=False):
    import torch
    T, E = SMALL["tokens"], SMALL["experts"]
    El = E // world
    full = of.qwen3_moe_graph(**SMALL)
    host = llama_inputs(full, T, seed=5)
    if skew:  # route most tokens to rank 0's experts (unbalanced receive counts)
        for name in host:
            if name.endswith("router.w"):
                host[name][:, :El] += 0.5
    rng = np.random.default_rng(world)
    xs = [np.ascontiguousarray(host["x"] + rng.uniform(-0.5, 0.5, host["x"].shape).astype(np.float32) * r)
          for r in range(world)]
    desc = of.qwen3_moe_graph(**SMALL, ep=world)
    comms = of.Comm.virtual(world, 0, 1 << 16)
    sessions, keep, outs = [], [], []
    for r in range(world):
        g = of.build_graph(desc)
        sess = of.Session(g, of.partition(g, RULES), {"lanes": 3}, comms[r])
        k = {}
        for t in g.description["tensors"]:
            name = t["name"]
            if t["role"] == "output":
                shape = list(t["shape"])
                k[name] = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
                outs.append((r, name, k[name]))
            elif t["role"] in ("input", "weight"):
                arr = xs[r] if name == "x" else host[name]
                if name.startswith("layer") and ".experts." in name:
                    arr = arr[r * El:(r + 1) * El]
                x = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
                if t.get("dtype") == "bf16":
                    x = x.to(torch.bfloat16)
                k[name] = x
            else:
                continue
            sess.bind(name, k[name])
        sessions.append(sess)
        keep.append(k)
    of.Session.link_virtual(sessions, 256 << 20)
    streams = [torch.cuda.Stream() for _ in range(world)]
    torch.cuda.synchronize()
    for r in range(world):
        sessions[r].prepare(strategy, streams[r])
    torch.cuda.synchronize()
    for _ in range(repeats):
        for r in range(world):
            sessions[r].run(strategy, streams[r])
    torch.cuda.synchronize()
    for c in comms:
        assert c.window_error() == 0
    got = {}
    for r, name, t in outs:
        got[(r, name)] = t.float().cpu().numpy()
    want = [oracle.evaluate(full, T, dict(host, x=xs[r]), exact=False) for r in range(world)]
    return got, want, sessions


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("strategy", [{"name": "sequential"}, {"name": "dbo", "align": 128}])
def test_ep_layer_vs_oracle(cuda, world, strategy):
    got, want, sessions = run_ep(world, strategy)
    for r in range(world):
        for name, w in want[r].items():
            assert rel_err(got[(r, name)], w) < 2e-2, (r, name)
    assert sessions[0].stats()["last"]["copied_elements"] == 0


def test_ep_skewed_routing(cuda):
    got, want, _ = run_ep(4, {"name": "dbo", "align": 128}, skew=True)
    for r in range(4):
        for name, w in want[r].items():
            assert rel_err(got[(r, name)], w) < 2e-2, (r, name)
