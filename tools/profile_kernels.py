"""Run each hot kernel once on its Llama-3-8B bench shape (for ncu captures):
  gemm (qkv 8192x6144x4096, gate_up+SiLU 8192x28672x4096), prefill attention
  (8 x 1024 tokens, 32/8 heads), paged decode attention (512 x 4K), add_rmsnorm,
  Qwen3 MoE expert FFN (dispatch, grouped gate_up / down, combine).
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
if which == "proj":  # the four Llama-3-8B projections at TP=1 (bench roofline shapes)
    gemm(T, H, 6144), gemm(T, H, 4096), gemm(T, H, 28672), gemm(T, 14336, H)
if which == "splitk":  # decode nano-batch down projection (S = 4 split-K) and decode O
    gemm(256, 14336, H), gemm(512, 4096, 6144)
if which == "proj_tp8":  # per-rank shapes at TP=8
    gemm(T, H, 768), gemm(T, 512, H), gemm(T, H, 3584), gemm(T, 1792, H)
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
if which in ("all", "moe"):
    # Qwen3-30B-A3B expert FFN: 8192 tokens, 128 experts, top-8, H 2048, moe_inter 768
    import json
    E, k, Hm, MI = 128, 8, 2048, 768
    ids = torch.argsort(torch.rand(T, E, device=dev), dim=1)[:, :k].contiguous()
    x = torch.randn(T, Hm, device=dev).to(torch.bfloat16)
    tens = [{"name": "x", "shape": [T, Hm], "dtype": "bf16", "role": "input"},
            {"name": "ids", "shape": [T, k], "dtype": "i64", "role": "input"},
            {"name": "wgu", "shape": [E, Hm, 2 * MI], "dtype": "bf16", "role": "weight", "batch": "replicated"},
            {"name": "wd", "shape": [E, MI, Hm], "dtype": "bf16", "role": "weight", "batch": "replicated"},
            {"name": "w", "shape": [T, k], "dtype": "f32", "role": "input"},
            {"name": "xd", "shape": [T, k * Hm], "dtype": "bf16"},
            {"name": "slot", "shape": [T, k], "dtype": "i64"},
            {"name": "hd", "shape": [T, k * MI], "dtype": "bf16"},
            {"name": "yd", "shape": [T, k * Hm], "dtype": "bf16"},
            {"name": "y", "shape": [T, Hm], "dtype": "bf16", "role": "output"}]
    prm = {"experts": E, "topk": k}
    ops = [{"name": "dispatch", "kind": "Custom", "inputs": ["x", "ids"], "outputs": ["xd", "slot"],
            "attrs": {"custom_name": "moe_dispatch", "params": prm}},
           {"name": "gate_up", "kind": "Custom", "inputs": ["xd", "ids", "wgu"], "outputs": ["hd"],
            "attrs": {"custom_name": "moe_gate_up", "params": prm}},
           {"name": "down", "kind": "Custom", "inputs": ["hd", "ids", "wd"], "outputs": ["yd"],
            "attrs": {"custom_name": "moe_down", "params": prm}},
           {"name": "combine", "kind": "Custom", "inputs": ["yd", "slot", "w"], "outputs": ["y"],
            "attrs": {"custom_name": "moe_combine", "params": prm}}]
    g = of.build_graph(json.dumps({"tensors": tens, "operators": ops}))
    s = of.Session(g, of.partition(g, []), {"lanes": 1})
    bind = {"x": x, "ids": ids, "w": torch.full((T, k), 1.0 / k, device=dev),
            "wgu": (torch.randn(E, Hm, 2 * MI, device=dev) / Hm ** 0.5).to(torch.bfloat16),
            "wd": (torch.randn(E, MI, Hm, device=dev) / MI ** 0.5).to(torch.bfloat16),
            "y": torch.empty(T, Hm, device=dev, dtype=torch.bfloat16)}
    for n_, t_ in bind.items():
        s.bind(n_, t_)
    for _ in range(2):
        s.run()
torch.cuda.synchronize()
print("done", which)
if which == "toy":  # BASELINE configs[0]: the fp32 toy decoder (exact stand-in MatMuls, short-sequence prefill)
    from pathlib import Path
    from paper_2605_21603_b200.workloads import llama_inputs
    root = Path(__file__).resolve().parent.parent
    desc = (root / "oracle" / "fixtures" / "toy_decoder_c1.json").read_text()
    host = llama_inputs(desc, 1024, seed=2026)
    g = of.build_graph(desc)
    s = of.Session(g, of.partition(g, []), {"lanes": 1})
    keep = {}
    for t in g.description["tensors"]:
        if t["role"] in ("input", "weight"):
            keep[t["name"]] = torch.from_numpy(host[t["name"]]).to(dev)
        elif t["role"] == "output":
            keep[t["name"]] = torch.empty(t["shape"], dtype=torch.float32, device=dev)
        else:
            continue
        s.bind(t["name"], keep[t["name"]])
    for _ in range(2):
        s.run()
    torch.cuda.synchronize()
