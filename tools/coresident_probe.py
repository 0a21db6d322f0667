"""Co-residency probe for NanoFlow decode (BASELINE configs[3] shapes): the
paged decode attention of one nano-batch (256 x 4K context) and the GEMMs of
the other (M = 256), each timed alone and both launched concurrently on two
streams, for the whole-GPU kernels and the co-resident (lane SM budget -1)
variants.  The co-resident variants (lane SM budget -1: 2/3-stage 2-CTA GEMM,
4/8-warp attention, OPF_COLOC_ATT / OPF_COLOC_STAGES) exist only in the library
of commit 7418aec: `git checkout 7418aec -- paper_2605_21603_b200/csrc` and
rebuild to reproduce.  Measured: no configuration beats running
the two whole-GPU kernels back to back.  Usage: python tools/coresident_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_21603_b200 import opflow as of  # noqa: E402

dev = torch.device("cuda:0")
B, ctx, page, nq, nkv, hd = 256, 4096, 16, 32, 8, 128
gen = torch.Generator(device=dev).manual_seed(3)


def session(tensors, ops, coloc, bind):
    desc = json.dumps({"tensors": tensors, "operators": ops})
    g = of.build_graph(desc)
    cfg = {"lanes": 1, "lane_sm_budget": [-1]} if coloc else {"lanes": 1}
    s = of.Session(g, of.partition(g, []), cfg)
    for k, v in bind.items():
        s.bind(k, v)
    return s


pages = B * ctx // page
kc = (torch.rand(pages, nkv, page, hd, device=dev, generator=gen) * 2 - 1).to(torch.bfloat16)
vc = (torch.rand(pages, nkv, page, hd, device=dev, generator=gen) * 2 - 1).to(torch.bfloat16)
qkv = (torch.rand(B, (nq + 2 * nkv) * hd, device=dev, generator=gen) * 2 - 1).to(torch.bfloat16)
table = torch.randperm(pages, device=dev, generator=gen).view(B, -1).to(torch.int64)
pos = torch.full((B,), ctx - 1, dtype=torch.int64, device=dev)
att_out = torch.empty(B, nq * hd, dtype=torch.bfloat16, device=dev)
att_t = [{"name": "qkv", "shape": list(qkv.shape), "dtype": "bf16", "role": "input"},
         {"name": "kc", "shape": list(kc.shape), "dtype": "bf16", "role": "weight", "batch": "replicated"},
         {"name": "vc", "shape": list(vc.shape), "dtype": "bf16", "role": "weight", "batch": "replicated"},
         {"name": "bt", "shape": list(table.shape), "dtype": "i64", "role": "input"},
         {"name": "pos", "shape": [B], "dtype": "i64", "role": "input"},
         {"name": "o", "shape": list(att_out.shape), "dtype": "bf16", "role": "output"}]
att_op = [{"name": "a", "kind": "Custom", "inputs": ["qkv", "kc", "vc", "bt", "pos"], "outputs": ["o"],
           "attrs": {"custom_name": "attn_decode",
                     "params": {"heads": nq, "kv_heads": nkv, "head_dim": hd, "page_size": page, "kv_layout": 1}}}]
att_bind = {"qkv": qkv, "kc": kc, "vc": vc, "bt": table, "pos": pos, "o": att_out}

GEMMS = {"qkv": (4096, 6144), "o": (4096, 4096), "gate_up": (4096, 28672), "down": (14336, 4096)}
gem_t, gem_op, gem_bind = [], [], {}
for name, (K, N) in GEMMS.items():
    a = (torch.rand(B, K, device=dev, generator=gen) * 2 - 1).to(torch.bfloat16)
    w = ((torch.rand(K, N, device=dev, generator=gen) * 2 - 1) / K ** 0.5).to(torch.bfloat16)
    c = torch.empty(B, N, dtype=torch.bfloat16, device=dev)
    gem_t += [{"name": f"{name}.a", "shape": [B, K], "dtype": "bf16", "role": "input"},
              {"name": f"{name}.w", "shape": [K, N], "dtype": "bf16", "role": "weight", "batch": "replicated"},
              {"name": f"{name}.c", "shape": [B, N], "dtype": "bf16", "role": "output"}]
    gem_op += [{"name": name, "kind": "MatMul", "inputs": [f"{name}.a", f"{name}.w"], "outputs": [f"{name}.c"]}]
    gem_bind.update({f"{name}.a": a, f"{name}.w": w, f"{name}.c": c})


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for mode in ("whole", "coloc"):
    co = mode == "coloc"
    att = session(att_t, att_op, co, att_bind)
    gem = session(gem_t, gem_op, co, gem_bind)
    res[f"{mode}.attn_ms"] = timed(lambda: att.run(None, torch.cuda.current_stream()))
    res[f"{mode}.gemms_ms"] = timed(lambda: gem.run(None, torch.cuda.current_stream()))

    def both():
        cur = torch.cuda.current_stream()
        s0.wait_stream(cur)
        s1.wait_stream(cur)
        att.run(None, s0)
        gem.run(None, s1)
        cur.wait_stream(s0)
        cur.wait_stream(s1)
    res[f"{mode}.both_ms"] = timed(both)
    # per-op GEMM times (each alone)
    for name in GEMMS:
        g1 = session([t for t in gem_t if t["name"].startswith(name + ".")],
                     [o for o in gem_op if o["name"] == name], co,
                     {k: v for k, v in gem_bind.items() if k.startswith(name + ".")})
        res[f"{mode}.{name}_ms"] = timed(lambda: g1.run(None, torch.cuda.current_stream()))
    del att, gem
for k in res:
    res[k] = round(res[k], 4)
kv = 2.0 * B * ctx * nkv * hd * 2
res["whole.attn_gbs"] = round(kv / res["whole.attn_ms"] / 1e6, 1)
res["coloc.attn_gbs"] = round(kv / res["coloc.attn_ms"] / 1e6, 1)
res["env"] = {k: v for k, v in os.environ.items() if k.startswith("OPF_COLOC")}
print(json.dumps(res))
