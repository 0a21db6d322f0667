"""Run each hot kernel once on its Llama-3-8B bench shape (for ncu captures):
  gemm (qkv 8192x6144x4096, gate_up+SiLU 8192x28672x4096), prefill attention
  (8 x 1024 tokens, 32/8 heads), paged decode attention (512 x 4K), add_rmsnorm.
Usage: ncu --set full -k regex:<kernel> python tools/profile_kernels.py [which]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_21603_b200 import opflow as of  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = torch.device("cuda:0")
T, H = 8192, 4096


def gemm(m, k, n, silu=False):
    import json
    ops = [{"name": "mm", "kind": "MatMul", "inputs": ["a", "w"], "outputs": ["c" if not silu else "gu"]}]
    tens = [{"name": "a", "shape": [m, k], "dtype": "bf16", "role": "input"},
            {"name": "w", "shape": [k, n], "batch": "replicated", "dtype": "bf16", "role": "weight"}]
    if silu:
        tens += [{"name": "gu", "shape": [m, n], "dtype": "bf16"},
                 {"name": "c", "shape": [m, n // 2], "dtype": "bf16", "role": "output"}]
        ops.append({"name": "act", "kind": "Custom", "inputs": ["gu"], "outputs": ["c"],
                    "attrs": {"custom_name": "silu_mul"}})
    else:
        tens.append({"name": "c", "shape": [m, n], "dtype": "bf16", "role": "output"})
    g = of.build_graph(json.dumps({"tensors": tens, "operators": ops}))
    s = of.Session(g, of.partition(g, []), {"lanes": 1})
    a = torch.randn(m, k, device=dev).to(torch.bfloat16)
    w = (torch.randn(k, n, device=dev) / k ** 0.5).to(torch.bfloat16)
    c = torch.empty(m, n // 2 if silu else n, device=dev, dtype=torch.bfloat16)
    s.bind("a", a), s.bind("w", w), s.bind("c", c)
    for _ in range(2):
        s.run()
    torch.cuda.synchronize()


if which in ("all", "gemm"):
    gemm(T, H, 6144)
if which in ("all", "gemm_silu"):
    gemm(T, H, 28672, silu=True)
if which in ("all", "prefill"):
    qkv = torch.randn(T, 48 * 128, device=dev).to(torch.bfloat16)
    out = torch.empty(T, 32 * 128, device=dev, dtype=torch.bfloat16)
    op = {"name": "a", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "attn_prefill", "params": {"heads": 32, "kv_heads": 8, "head_dim": 128,
                                                               "seq_len": 1024}}}
    for _ in range(2):
        of.launch(op, [qkv], [out], T)
if which in ("all", "decode"):
    B, ctx, page = 512, 4096, 16
    pages = B * ctx // page
    kc = torch.randn(pages, page, 8, 128, device=dev).to(torch.bfloat16)
    vc = torch.randn(pages, page, 8, 128, device=dev).to(torch.bfloat16)
    table = torch.randperm(pages, device=dev).view(B, -1)
    pos = torch.full((B,), ctx - 1, dtype=torch.int64, device=dev)
    qkv = torch.randn(B, 48 * 128, device=dev).to(torch.bfloat16)
    out = torch.empty(B, 32 * 128, device=dev, dtype=torch.bfloat16)
    op = {"name": "d", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "attn_decode", "params": {"heads": 32, "kv_heads": 8, "head_dim": 128,
                                                              "page_size": page}}}
    for _ in range(2):
        of.launch(op, [qkv, kc, vc, table, pos], [out], B)
if which in ("all", "norm"):
    x = torch.randn(T, H, device=dev).to(torch.bfloat16)
    r = torch.randn(T, H, device=dev).to(torch.bfloat16)
    gm = torch.ones(H, device=dev).to(torch.bfloat16)
    s_, y = torch.empty_like(x), torch.empty_like(x)
    op = {"name": "n", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "add_rmsnorm", "params": {"eps": 1e-5}}}
    for _ in range(2):
        of.launch(op, [x, r, gm], [s_, y], T)
torch.cuda.synchronize()
print("done", which)
