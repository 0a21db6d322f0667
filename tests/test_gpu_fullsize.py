"""GPU parity at BASELINE.json's bench shapes (not just small cases): one
Llama-3-8B-shaped prefill layer (8 x 1024 tokens), one decode layer (512
sequences x 4K context, HND pages) and one Qwen3-30B-A3B MoE layer (8192
tokens), each through the engine's overlapped schedule, against a plain
PyTorch fp32 reference of the same graph (tests/torch_ref.py).  Tolerance:
bf16 normwise relative error <= 2e-2 (north star)."""
import json

import pytest

from paper_2605_21603_b200 import opflow as of
from torch_ref import evaluate

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("built")]

LLAMA = dict(hidden=4096, heads=32, kv_heads=8, head_dim=128, inter=14336)
QWEN3 = dict(hidden=2048, heads=32, kv_heads=4, head_dim=128, experts=128, topk=8, moe_inter=768)


def _bind_random(desc, rows, seed, special=None):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    d = json.loads(desc)
    out = {}
    for t in d["tensors"]:
        if t["role"] not in ("input", "weight"):
            continue
        n, shape = t["name"], list(t["shape"])
        if t.get("batch", "batched") == "batched" and t["role"] == "input":
            shape[0] = rows
        if special and n in special:
            out[n] = special[n]
            continue
        if t.get("dtype") == "i64":
            continue
        if n.endswith("norm.w"):
            x = 1.0 + 0.1 * (torch.rand(shape, device="cuda", generator=g) - 0.5)
        elif t["role"] == "weight":
            fan_in = shape[-2] if len(shape) == 3 else shape[0]
            x = (torch.rand(shape, device="cuda", generator=g) * 2 - 1) / fan_in ** 0.5
        else:
            x = torch.rand(shape, device="cuda", generator=g) * 2 - 1
        out[n] = x.to(torch.bfloat16)
    return out


def _run(desc, rows, bind, spec, rules=()):
    import torch
    gr = of.build_graph(desc)
    sess = of.Session(gr, of.partition(gr, list(rules)), {"lanes": 3})
    for n, v in bind.items():
        sess.bind(n, v)
    outs = {}
    for t in json.loads(desc)["tensors"]:
        if t["role"] == "output":
            shape = list(t["shape"])
            shape[0] = rows
            outs[t["name"]] = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
            sess.bind(t["name"], outs[t["name"]])
    sess.run(spec)
    torch.cuda.synchronize()
    return outs


def _check(got, want):
    for k in want:
        g, w = got[k].float(), want[k].float()
        err = ((g - w).norm() / w.norm()).item()
        print(f"{k}: normwise rel err {err:.3e}")
        assert err < 2e-2, (k, err)


def test_llama8b_prefill_layer_full_size(cuda):
    import torch
    T, S = 8192, 1024
    desc = of.llama_graph(layers=1, tokens=T, seq_len=S, dtype="bf16", **LLAMA)
    pos = (torch.arange(T, device="cuda") % S).to(torch.int64)
    bind = _bind_random(desc, T, 11, {"positions": pos})
    want = evaluate(desc, T, bind)
    got = _run(desc, T, bind, {"name": "split_overlap", "n_microbatches": 2, "align": S, "lane_mode": "ubatch"})
    _check(got, want)


def test_llama8b_decode_layer_full_size(cuda):
    import torch
    B, ctx, page = 512, 4096, 16
    desc = of.llama_decode_graph(layers=1, tokens=B, ctx_len=ctx, page_size=page, dtype="bf16", kv_layout=1,
                                 **LLAMA)
    g = torch.Generator(device="cuda").manual_seed(5)
    pages = B * ctx // page
    lens = torch.randint(1, ctx, (B,), device="cuda", generator=g).to(torch.int64)
    special = {"positions": lens,
               "block_table": torch.randperm(pages, device="cuda", generator=g).view(B, -1).to(torch.int64)}
    bind = _bind_random(desc, B, 12, special)
    for n in list(bind):
        if n.endswith("_cache"):  # KV cache content ~U(-1, 1)
            bind[n] = (torch.rand(bind[n].shape, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    want = evaluate(desc, B, bind)
    got = _run(desc, B, bind, {"name": "split_overlap", "n_microbatches": 2, "lane_mode": "ubatch"},
               [of.PartitionRule.by_func("attn_decode")])
    _check(got, want)


def test_qwen3_moe_layer_full_size(cuda):
    import torch
    T, S = 8192, 1024
    desc = of.qwen3_moe_graph(layers=1, tokens=T, seq_len=S, dtype="bf16", ep=1, **QWEN3)
    pos = (torch.arange(T, device="cuda") % S).to(torch.int64)
    bind = _bind_random(desc, T, 13, {"positions": pos})
    want = evaluate(desc, T, bind)
    R = of.PartitionRule
    rules = [R.by_module("layer*.attn"), R.by_module("layer*.moe.dispatch"), R.by_module("layer*.moe.experts"),
             R.by_module("layer*.moe.combine")]
    got = _run(desc, T, bind, {"name": "dbo", "align": S}, rules)
    _check(got, want)
