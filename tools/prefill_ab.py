"""Prefill leg (Llama-3-8B-shaped, 8 x 1024 tokens, TP=1) for same-box A/B
runs: OPF_LIB=<variant .so> python tools/prefill_ab.py [layers].  Prints one
JSON line of per-strategy ms/step (interleaved median, after a soak)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_21603_b200 import opflow as of  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
T, S = 8192, 1024
dev = torch.device("cuda:0")
desc = of.llama_graph(layers=L, tokens=T, seq_len=S, tp=1, dtype="bf16", **bench.LLAMA)
extra = json.loads(os.environ.get("SESSION_CFG", "{}"))  # e.g. {"fuse_addnorm": false}
g, plan, sess, bufs = bench.build_session(of, desc, [], dev, None, seed=1234, extra_cfg=extra)
pos = (torch.arange(T, device=dev) % S).to(torch.int64)
sess.bind("positions", pos)
cands = {"sequential": {"name": "sequential"},
         "nanoflow_u2": {"name": "split_overlap", "n_microbatches": 2, "align": S, "lane_mode": "ubatch"}}
res = bench.time_candidates(torch, sess, cands, 5, 3, torch.cuda.current_stream(dev), 1)
print(json.dumps({"lib": os.environ.get("OPF_LIB", "default"), "cfg": extra, "layers": L,
                  "ms_per_layer": {k: round(v / L, 4) for k, v in res.items()},
                  "launches": sess.stats()["last"]["launches"]}))
