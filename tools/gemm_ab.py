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
out = {}
for (m, n, k) in SHAPES:
    d = json.dumps({"tensors": [{"name": "a", "shape": [m, k], "dtype": "bf16", "role": "input"},
                                {"name": "w", "shape": [k, n], "batch": "replicated", "dtype": "bf16", "role": "weight"},
                                {"name": "c", "shape": [m, n], "dtype": "bf16", "role": "output"}],
                    "operators": [{"name": "mm", "kind": "MatMul", "inputs": ["a", "w"], "outputs": ["c"]}]})
    g = of.build_graph(d)
    s = of.Session(g, of.partition(g, []), {"lanes": 1})
    a = torch.randn(m, k, device=dev).to(torch.bfloat16)
    w = (torch.randn(k, n, device=dev) / k ** 0.5).to(torch.bfloat16)
    c = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    s.bind("a", a), s.bind("w", w), s.bind("c", c)
    for _ in range(5):
        s.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        s.run()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    out[f"{m}x{n}x{k}"] = [round(us, 1), _lib.lib().opf_gemm_splits(m, n, k, 0),
                           round(2.0 * m * n * k / us / 1e6, 1)]
    del s
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("OPF_GEMM")}, "us_splits_tflops": out}))
