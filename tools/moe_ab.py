"""The bench's MoE leg (BASELINE configs[4], Qwen3-30B-A3B layer, 8192 tokens)
alone, for same-box A/B runs (OPF_LIB=<variant .so>).  Prints one JSON line."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_21603_b200 import opflow as of  # noqa: E402

a = argparse.Namespace(seq_len=1024, moe_layers=1, tokens=8192, steps=20, warmup=5)
dev = torch.device("cuda:0")
r = bench.run_moe(of, torch, dev, a, 0, 1, torch.cuda.current_stream(dev))
print(json.dumps({"lib": os.environ.get("OPF_LIB", "default"), "strategies_ms": r["strategies_ms"],
                  "per_op": r["roofline"]["per_op"]}))
