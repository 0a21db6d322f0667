"""Time the tcgen05 GEMM on the Llama-3-8B projection shapes (and a few more)
with CUDA events; OPF_GEMM=1sm|2sm|auto selects the kernel variant."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_21603_b200 import opflow as of  # noqa: E402

T = int(os.environ.get("T", 8192))
shapes = {"qkv": (T, 4096, 6144), "o": (T, 4096, 4096), "gate_up": (T, 4096, 28672),
          "down": (T, 14336, 4096), "tp8_o": (T, 512, 4096), "tp8_qkv": (T, 4096, 768),
          "decode_gate_up": (512, 4096, 28672)}
dev = torch.device("cuda:0")
ach, rows = bench.gemm_roofline(of, torch, dev, shapes, reps=30)
print(json.dumps({"mode": os.environ.get("OPF_GEMM", "auto"), "weighted_tflops": round(ach, 1),
                  "rows": rows}))
