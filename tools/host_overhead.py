"""Host-side cost of one Session.run (spec parse, plan-cache lookup, graph
launch) on the MoE layer session, GPU work queued asynchronously."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_21603_b200 import opflow as of  # noqa: E402

dev = torch.device("cuda:0")
Q = bench.QWEN3
T, S = 8192, 1024
desc = of.qwen3_moe_graph(layers=1, tokens=T, seq_len=S, dtype="bf16", ep=1, **Q)
R = of.PartitionRule
rules = [R.by_module("layer*.attn"), R.by_module("layer*.moe.dispatch"), R.by_module("layer*.moe.experts"),
         R.by_module("layer*.moe.combine")]
g, plan, sess, bufs = bench.build_session(of, desc, rules, dev, None, seed=1)
pos = (torch.arange(T, device=dev) % S).to(torch.int64)
sess.bind("positions", pos)
seq = {"name": "sequential"}
dbo = {"name": "dbo", "align": S}
auto = {"name": "auto", "reps": 3, "candidates": [seq, dbo]}
out = {}
def run(spec):
    if isinstance(spec, str):  # exact spec text (the key auto's choice is cached under)
        of.check(of.lib().opf_session_run(sess._h, spec.encode(), None))
    else:
        sess.run(spec)


for name, spec in [("sequential", seq), ("dbo", dbo), ("auto", auto), ("seq_compact", '{"name":"sequential"}'),
                   ("sequential_again", seq)]:
    for _ in range(5):
        run(spec)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        run(spec)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out[name] = {"host_us_per_run": round((t1 - t0) / 50 * 1e6, 1), "wall_us_per_run": round((t2 - t0) / 50 * 1e6, 1)}
print(json.dumps(out))
