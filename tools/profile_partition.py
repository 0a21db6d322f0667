"""One launch each of the two NanoFlow decode partners at their partitioned SM
budgets and at the full GPU, for ncu counter captures (dram throughput of the
paged attention, tensor-pipe activity of the half-batch GEMMs):
  ncu --set full -k regex:"decode_t|gemm_tc2" python tools/profile_partition.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_21603_b200 import opflow as of  # noqa: E402

dev = torch.device("cuda:0")
B, ctx, page, nq, nkv, hd = 512, 4096, 16, 32, 8, 128
g = torch.Generator(device=dev).manual_seed(3)
pages = B * ctx // page
kc = torch.rand(pages, nkv, page, hd, device=dev, generator=g).to(torch.bfloat16)
vc = torch.rand(pages, nkv, page, hd, device=dev, generator=g).to(torch.bfloat16)
table = torch.randperm(pages, device=dev, generator=g).view(B, -1)
pos = torch.full((B,), ctx - 1, dtype=torch.int64, device=dev)
qkv = torch.randn(B, (nq + 2 * nkv) * hd, device=dev).to(torch.bfloat16)
out = torch.empty(B, nq * hd, device=dev, dtype=torch.bfloat16)
op = {"name": "d", "kind": "Custom", "inputs": [], "outputs": [],
      "attrs": {"custom_name": "attn_decode",
                "params": {"heads": nq, "kv_heads": nkv, "head_dim": hd, "page_size": page, "kv_layout": 1}}}
for sms in (148, 108):  # attention alone at the full GPU and at its NanoFlow share
    of.launch(op, [qkv, kc, vc, table, pos], [out], B, max_ctas=sms)
torch.cuda.synchronize()
half = B // 2
for sms in (148, 40):  # half-batch gate_up GEMM at the full GPU and at its NanoFlow share
    d = json.dumps({"tensors": [{"name": "a", "shape": [half, 4096], "dtype": "bf16", "role": "input"},
                                {"name": "w", "shape": [4096, 28672], "batch": "replicated", "dtype": "bf16",
                                 "role": "weight"},
                                {"name": "c", "shape": [half, 28672], "dtype": "bf16", "role": "output"}],
                    "operators": [{"name": "mm", "kind": "MatMul", "inputs": ["a", "w"], "outputs": ["c"]}]})
    gg = of.build_graph(d)
    s = of.Session(gg, of.partition(gg, []), {"lanes": 1, "lane_sm_budget": [sms]})
    a = torch.randn(half, 4096, device=dev).to(torch.bfloat16)
    w = (torch.randn(4096, 28672, device=dev) / 64).to(torch.bfloat16)
    c = torch.empty(half, 28672, device=dev, dtype=torch.bfloat16)
    s.bind("a", a), s.bind("w", w), s.bind("c", c)
    s.run()
    torch.cuda.synchronize()
print("done")
