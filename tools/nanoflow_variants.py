"""NanoFlow split variants at the bench shape (8 layers, 8192 tokens, TP=1): ms per layer."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_21603_b200 import opflow as of
L, T, S = 8, 8192, 1024
dev = torch.device("cuda:0")
desc = of.llama_graph(layers=L, tokens=T, seq_len=S, tp=1, dtype="bf16", **bench.LLAMA)
g, plan, sess, bufs = bench.build_session(of, desc, [], dev, None, seed=1234)
sess.bind("positions", (torch.arange(T, device=dev) % S).to(torch.int64))
u = {"lane_mode": "ubatch", "align": S}
cands = {"sequential": {"name": "sequential"},
         "u2": dict(u, name="split_overlap", n_microbatches=2),
         "u3": dict(u, name="split_overlap", n_microbatches=3),
         "u4": dict(u, name="split_overlap", n_microbatches=4),
         "s5_3": dict(u, name="split_overlap", sizes=[5120, 3072]),
         "s6_2": dict(u, name="split_overlap", sizes=[6144, 2048]),
         "u2_b74": dict(u, name="split_overlap", n_microbatches=2, lane_sm_budget=[74, 74, 74]),
         "u2_b112": dict(u, name="split_overlap", n_microbatches=2, lane_sm_budget=[112, 112, 112])}
res = bench.time_candidates(torch, sess, cands, 5, 3, torch.cuda.current_stream(dev), 1)
print(json.dumps({k: round(v / L, 4) for k, v in res.items()}))
