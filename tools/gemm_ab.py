"""A/B timing of the tcgen05 GEMM on decode / TP-sharded shapes through a
one-op Session (engine workspace, so split-K is available).  Run it twice
with different OPF_GEMM_* env settings in the same gpurun call.
Prints one JSON line {shape: us}."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_21603_b200 import _lib, opflow as of  # noqa: E402

SHAPES = [(512, 6144, 4096), (512, 4096, 4096), (512, 28672, 4096), (512, 4096, 14336),
          (256, 6144, 4096), (256, 4096, 4096), (256, 28672, 4096), (256, 4096, 14336),
          (8192, 768, 4096), (8192, 4096, 512), (8192, 3584, 4096), (8192, 4096, 1792),
          (8192, 6144, 4096), (8192, 4096, 4096), (8192, 28672, 4096), (8192, 4096, 14336)]
dev = torch.device("cuda:0")
import bench  # noqa: E402
if os.environ.get("AB_SHAPES"):
    SHAPES = [tuple(int(v) for v in x.split("x")) for x in os.environ["AB_SHAPES"].split(",")]
out = {}
stream = torch.cuda.current_stream(dev)
for (m, n, k) in SHAPES:
    # device time: 8 launches back to back in one CUDA graph, rotated A / W / C
    a = torch.randn(m, k, device=dev).to(torch.bfloat16)
    w = (torch.randn(k, n, device=dev) / k ** 0.5).to(torch.bfloat16)
    c = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    op = {"name": "mm", "kind": "MatMul", "inputs": ["a", "w"], "outputs": ["c"]}
    ms = bench.graph_reps_ms(of, torch, dev, stream, [("a", a, "input"), ("w", w, "weight"), ("c", c, "output")],
                             op, shared=(), reps=8)
    us = ms * 1e3
    out[f"{m}x{n}x{k}"] = [round(us, 1), _lib.lib().opf_gemm_splits(m, n, k, 0),
                           round(2.0 * m * n * k / us / 1e6, 1)]
print(json.dumps({"lib": os.environ.get("OPF_LIB", "default"),
                  "env": {k: v for k, v in os.environ.items() if k.startswith("OPF_GEMM")}, "us_splits_tflops": out}))
