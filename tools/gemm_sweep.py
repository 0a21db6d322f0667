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
          "decode_gate_up": (512, 4096, 28672), "tp8_gate_up": (T, 4096, 3584),
          "tp8_down": (T, 1792, 4096), "tp2_qkv": (T, 4096, 3072), "tp2_o": (T, 2048, 4096),
          "tp4_o": (T, 1024, 4096), "tp4_qkv": (T, 4096, 1536)}
dev = torch.device("cuda:0")
ach, rows = bench.gemm_roofline(of, torch, dev, shapes, reps=30)
cublas = {}
for name, (m, k, n) in shapes.items():
    a = torch.randn(m, k, device=dev, dtype=torch.bfloat16)
    w = torch.randn(k, n, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(a, w)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30):
        torch.matmul(a, w)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    cublas[name] = round(2.0 * m * n * k / ms / 1e9, 1)
for r in rows:
    r["cublas_tflops"] = cublas[r["gemm"]]
print(json.dumps({"mode": os.environ.get("OPF_GEMM", "auto"), "weighted_tflops": round(ach, 1),
                  "rows": rows}))
