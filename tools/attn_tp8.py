"""Per-rank attention kernels at the north-star TP=2/4/8 shapes on one B200:
prefill (8 x 1024 tokens, 4 q / 1 kv heads per rank, causal) and paged decode
(512 seqs x 4K context, 4 q / 1 kv heads per rank, random block table), next to
the TP=1 shapes.  Prints one JSON line (us, TFLOP/s or GB/s)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_21603_b200 import opflow as of  # noqa: E402
import bench  # noqa: E402

dev = torch.device("cuda:0")
hd, page = 128, 16
res = {}


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for tp in [int(x) for x in os.environ.get("TPS", "1 8").split()]:
    nq, nkv = 32 // tp, 8 // tp
    S, seqs = 1024, 8
    rows = S * seqs
    t = (torch.rand(rows, (nq + 2 * nkv) * hd, device=dev) * 2 - 1).to(torch.bfloat16)
    out = torch.empty(rows, nq * hd, dtype=torch.bfloat16, device=dev)
    op = {"name": "a", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "attn_prefill",
                    "params": {"heads": nq, "kv_heads": nkv, "head_dim": hd, "seq_len": S}}}
    ms = timed(lambda: of.launch(op, [t], [out], rows))
    fl = 4 * (S * (S + 1) / 2) * hd * nq * seqs
    res[f"prefill_tp{tp}"] = {"us": round(ms * 1e3, 1), "tflops": round(fl / ms / 1e9, 1)}
    B, ctx = int(os.environ.get("DEC_B", 512)), 4096
    pages = B * ctx // page
    g = torch.Generator(device=dev).manual_seed(3)
    kc = torch.rand(pages, nkv, page, hd, device=dev, generator=g).to(torch.bfloat16)
    vc = torch.rand(pages, nkv, page, hd, device=dev, generator=g).to(torch.bfloat16)
    table = torch.randperm(pages, device=dev, generator=g).view(B, -1)
    pos = torch.full((B,), ctx - 1, dtype=torch.int64, device=dev)
    qkv = torch.randn(B, (nq + 2 * nkv) * hd, device=dev).to(torch.bfloat16)
    o2 = torch.empty(B, nq * hd, device=dev, dtype=torch.bfloat16)
    dop = {"name": "d", "kind": "Custom", "inputs": [], "outputs": [],
           "attrs": {"custom_name": "attn_decode",
                     "params": {"heads": nq, "kv_heads": nkv, "head_dim": hd, "page_size": page, "kv_layout": 1}}}
    dop.update(inputs=["qkv", "k_cache", "v_cache", "block_table", "positions"], outputs=["out"])
    ms = bench.graph_reps_ms(of, torch, dev, torch.cuda.current_stream(dev),
                             [("qkv", qkv, "input"), ("k_cache", kc, "weight"), ("v_cache", vc, "weight"),
                              ("block_table", table, "input"), ("positions", pos, "input"), ("out", o2, "output")],
                             dop, shared=("k_cache", "v_cache", "block_table", "positions"), reps=4)
    kvb = 2.0 * B * ctx * nkv * hd * 2
    res[f"decode_tp{tp}"] = {"us": round(ms * 1e3, 1), "gbs": round(kvb / ms / 1e6, 1)}
    del kc, vc
    torch.cuda.empty_cache()
print(json.dumps(res))
