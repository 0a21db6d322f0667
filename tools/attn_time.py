#!/usr/bin/env python3
"""Time the prefill attention implementations at the bench shape (8 x 1024
tokens, 32 q / 8 kv heads, hd 128) with CUDA events; report causal TFLOP/s
(4 * S^2/2 * hd * heads * seqs flops)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2605_21603_b200 import opflow as of  # noqa: E402

S = int(os.environ.get("S", 1024))
seqs = int(os.environ.get("SEQS", 8))
nq, nkv, hd = 32, 8, 128
rows = S * seqs
t = (torch.rand(rows, (nq + 2 * nkv) * hd, device="cuda") * 2 - 1).to(torch.bfloat16)
flops = 4 * (S * (S + 1) / 2) * hd * nq * seqs
res = {}
for impl, name in ((0, "tcgen05"), (1, "fa2_mma_sync")):
    op = {"name": "a", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "attn_prefill",
                    "params": {"heads": nq, "kv_heads": nkv, "head_dim": hd, "seq_len": S, "impl": impl}}}
    out = torch.empty(rows, nq * hd, dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        of.launch(op, [t], [out], rows)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        of.launch(op, [t], [out], rows)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    res[name] = out.float()
    print(f"{name:14s} {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.1f} TFLOP/s")
d = (res["tcgen05"] - res["fa2_mma_sync"]).abs().max().item()
print("max |tcgen05 - fa2| =", d)
