"""In-situ per-kernel breakdown of one step (prefill | moe) (eager replay of the compiled plan
with CUDA events around every launch, OPF_TRACE_LAUNCHES=1): prefill
(Llama-3-8B-shaped layers, 8 x 1024 tokens) or decode (512 x 4K, HND pages).
Usage: python tools/step_breakdown.py [prefill|decode] [layers]"""
import collections
import json
import os
import sys

os.environ["OPF_TRACE_LAUNCHES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_21603_b200 import opflow as of  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "prefill"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dev = torch.device("cuda:0")
T, S = 8192, 1024
if which == "decode":
    B, ctx, page = 512, 4096, 16
    desc = of.llama_decode_graph(layers=L, tokens=B, ctx_len=ctx, page_size=page, dtype="bf16", kv_layout=1,
                                 kv_write=1, **bench.LLAMA)
    g = of.build_graph(desc)
    sess = of.Session(g, of.partition(g, []), {"lanes": 3})
    gen = torch.Generator(device=dev).manual_seed(1)
    pages = B * ctx // page
    kc = torch.rand(pages, 8, page, 128, device=dev, generator=gen).to(torch.bfloat16)
    vc = torch.rand(pages, 8, page, 128, device=dev, generator=gen).to(torch.bfloat16)
    keep = {}
    for t in g.description["tensors"]:
        n, shape = t["name"], t["shape"]
        if t["role"] not in ("input", "weight", "output") or (t["role"] == "output" and t.get("dtype") == "i64"):
            continue
        if n.endswith("k_cache"):
            x = kc
        elif n.endswith("v_cache"):
            x = vc
        elif n == "positions":
            x = torch.full((B,), ctx - 1, dtype=torch.int64, device=dev)
        elif n == "block_table":
            x = torch.randperm(pages, device=dev, generator=gen).view(B, -1)
        elif n == "slots":
            continue
        elif t["role"] == "output":
            x = torch.empty(shape, dtype=torch.bfloat16, device=dev)
        else:
            x = ((torch.rand(shape, device=dev, generator=gen) * 2 - 1) / (shape[0] ** 0.5 if t["role"] == "weight" else 1)).to(torch.bfloat16)
        keep[n] = x
        sess.bind(n, x)
    keep["slots"] = keep["block_table"][:, (ctx - 1) // page] * page + (ctx - 1) % page
    sess.bind("slots", keep["slots"])
elif which == "moe":
    desc = of.qwen3_moe_graph(layers=L, tokens=T, seq_len=S, dtype="bf16", ep=1, **bench.QWEN3)
else:
    desc = of.llama_graph(layers=L, tokens=T, seq_len=S, tp=1, dtype="bf16", **bench.LLAMA)
if which != "decode":
    g, plan, sess, bufs = bench.build_session(of, desc, [], dev, None, seed=1)
    sess.bind("positions", (torch.arange(T, device=dev) % S).to(torch.int64))
spec = {"name": "sequential"}
for _ in range(5):
    sess.run(spec)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    sess.run(spec)
e1.record()
torch.cuda.synchronize()
graph_ms = e0.elapsed_time(e1) / 10  # CUDA-graph replay of the same plan
tr = sess.trace()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in tr:
    key = e["name"].split(" u")[0]
    key = key.split(".", 1)[1] if key.startswith("layer") else key
    agg[key][0] += 1
    agg[key][1] += e["dur"] / 1e3
tot = sum(v[1] for v in agg.values())
span = (max(e["ts"] + e["dur"] for e in tr) - min(e["ts"] for e in tr)) / 1e3
rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
print(json.dumps({"which": which, "layers": L, "graph_replay_ms": round(graph_ms, 3), "span_ms": round(span, 3),
                  "sum_ms": round(tot, 3),
                  "per_kernel_ms_per_layer": {k: round(v[1] / L, 4) for k, v in rows}}, indent=1))
