"""NanoFlow decode overlap diagnostics (BASELINE configs[3] shape, a few layers):
per-dispatch eager trace of each schedule (lane, start, duration) and the two
overlapped kernels timed alone at reduced SM budgets.
Usage: python tools/decode_overlap.py [layers] [G ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_21603_b200 import opflow as of  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
GS = [int(x) for x in sys.argv[2:]] or [40]
B, ctx, page = 512, 4096, 16
H, nq, nkv, hd, I = 4096, 32, 8, 128, 14336
dev = torch.device("cuda:0")
nsm = torch.cuda.get_device_properties(dev).multi_processor_count
desc = of.llama_decode_graph(layers=L, tokens=B, ctx_len=ctx, page_size=page, hidden=H, heads=nq,
                             kv_heads=nkv, head_dim=hd, inter=I, dtype="bf16", kv_layout=1)
g = of.build_graph(desc)
sess = of.Session(g, of.partition(g, [of.PartitionRule.by_func("attn_decode")]), {"lanes": 3})
gen = torch.Generator(device=dev).manual_seed(5)
pages = B * ctx // page
kc = (torch.rand(pages, nkv, page, hd, device=dev, generator=gen) * 2 - 1).to(torch.bfloat16)
vc = (torch.rand(pages, nkv, page, hd, device=dev, generator=gen) * 2 - 1).to(torch.bfloat16)
keep = {}
for t in g.description["tensors"]:
    n, shape = t["name"], t["shape"]
    if t["role"] not in ("input", "weight", "output"):
        continue
    if n.endswith("k_cache"):
        x = kc
    elif n.endswith("v_cache"):
        x = vc
    elif n == "positions":
        x = torch.full((B,), ctx - 1, dtype=torch.int64, device=dev)
    elif n == "block_table":
        x = torch.randperm(pages, device=dev, generator=gen).view(B, -1).to(torch.int64)
    elif t["role"] == "output":
        x = torch.empty(shape, dtype=torch.bfloat16, device=dev)
    else:
        x = ((torch.rand(shape, device=dev, generator=gen) * 2 - 1) / (shape[0] ** 0.5 if t["role"] == "weight" else 1)).to(torch.bfloat16)
    keep[n] = x
    sess.bind(n, x)
specs = {"sequential": {"name": "sequential"},
         "nanoflow_u2": {"name": "split_overlap", "n_microbatches": 2, "lane_mode": "ubatch"},
         "nanoflow_class": {"name": "split_overlap", "n_microbatches": 2}}
for G in GS:
    specs[f"nanoflow_class_sm{G}"] = {"name": "split_overlap", "n_microbatches": 2, "lane_sm_budget": [G, nsm - G, 0]}
res = {}
for name, spec in specs.items():
    for _ in range(3):
        sess.run(spec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sess.run(spec)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    tr = sess.trace()
    res[name] = {"graph_ms": round(ms, 3),
                 "trace": [(d["name"][:40], d["tid"], round(d["ts"] / 1e3, 3), round(d["dur"] / 1e3, 3)) for d in tr]}
    print(f"== {name}: graph {ms:.3f} ms/step ({ms / L:.3f} per layer)")
    for row in res[name]["trace"][: 4 * 5]:
        print("   ", row)


def time_launch(op, ins, outs, rows, max_ctas, reps=20):
    for _ in range(3):
        of.launch(op, ins, outs, rows, max_ctas=max_ctas)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        of.launch(op, ins, outs, rows, max_ctas=max_ctas)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


half = B // 2
qkv = torch.randn(half, (nq + 2 * nkv) * hd, device=dev).to(torch.bfloat16)
out = torch.empty(half, nq * hd, device=dev, dtype=torch.bfloat16)
aop = {"name": "a", "kind": "Custom", "inputs": [], "outputs": [],
       "attrs": {"custom_name": "attn_decode", "params": {"heads": nq, "kv_heads": nkv, "head_dim": hd, "page_size": page,
                                                          "kv_layout": 1}}}
ins = [qkv, kc, vc, keep["block_table"][:half], keep["positions"][:half]]
kvb = 2.0 * half * ctx * nkv * hd * 2
print("attention (half batch) alone:")
for sms in [nsm, nsm - 24, nsm - 40, nsm - 56, 64, 48, 32]:
    ms = time_launch(aop, ins, [out], half, sms)
    print(f"   {sms:4d} SMs: {ms:.4f} ms  {kvb / ms / 1e6:.0f} GB/s")
print("GEMMs (half batch, M=256) via a 1-op session with lane budget:")
for (n_, k_, nn) in [("qkv", H, (nq + 2 * nkv) * hd), ("o", nq * hd, H), ("gate_up", H, 2 * I), ("down", I, H)]:
    d = json.dumps({"tensors": [{"name": "a", "shape": [half, k_], "dtype": "bf16", "role": "input"},
                                {"name": "w", "shape": [k_, nn], "batch": "replicated", "dtype": "bf16", "role": "weight"},
                                {"name": "c", "shape": [half, nn], "dtype": "bf16", "role": "output"}],
                    "operators": [{"name": "mm", "kind": "MatMul", "inputs": ["a", "w"], "outputs": ["c"]}]})
    row = []
    for sms in [nsm, 72, 56, 40, 24]:
        gg = of.build_graph(d)
        s = of.Session(gg, of.partition(gg, []), {"lanes": 1, "lane_sm_budget": [sms]})
        a = torch.randn(half, k_, device=dev).to(torch.bfloat16)
        w = (torch.randn(k_, nn, device=dev) / k_ ** 0.5).to(torch.bfloat16)
        c = torch.empty(half, nn, device=dev, dtype=torch.bfloat16)
        s.bind("a", a), s.bind("w", w), s.bind("c", c)
        for _ in range(3):
            s.run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            s.run()
        e1.record()
        torch.cuda.synchronize()
        row.append(f"{sms}:{e0.elapsed_time(e1) / 20 * 1e3:.1f}us")
    print(f"   {n_:8s}", " ".join(row))
json.dump(res, open("gpurun_out/decode_overlap.json", "w"))
