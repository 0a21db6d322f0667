"""Replay the bench's prefill (or decode) plan a few times and nothing else —
the command for a clean ncu launch list of the timed step:
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \\
      python tools/replay_step.py prefill 4 [strategy-json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_21603_b200 import opflow as of  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "prefill"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {"name": "sequential"}
dev = torch.device("cuda:0")
T, S = 8192, 1024
desc = of.llama_graph(layers=L, tokens=T, seq_len=S, tp=1, dtype="bf16", **bench.LLAMA)
g, plan, sess, bufs = bench.build_session(of, desc, [], dev, None, seed=1)
sess.bind("positions", (torch.arange(T, device=dev) % S).to(torch.int64))
for _ in range(3):
    sess.run(spec)
torch.cuda.synchronize()
