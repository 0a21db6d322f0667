"""Paged decode attention alone (512 x 4K, 32/8 heads, random block table) at
several SM budgets: achieved GB/s of algorithmic KV bytes.  The curve decides
whether NanoFlow can hand SMs to the GEMMs (OPF_LIB / OPF_DECODE for A/B)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_21603_b200 import opflow as of  # noqa: E402

B, ctx, page, nq, nkv, hd = 512, 4096, 16, 32, 8, 128
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(3)
pages = B * ctx // page
hnd = os.environ.get("DEC_LAYOUT", "hnd") == "hnd"
shape = (pages, nkv, page, hd) if hnd else (pages, page, nkv, hd)
kc = torch.rand(*shape, device=dev, generator=g).to(torch.bfloat16)
vc = torch.rand(*shape, device=dev, generator=g).to(torch.bfloat16)
table = torch.randperm(pages, device=dev, generator=g).view(B, -1)
pos = torch.full((B,), ctx - 1, dtype=torch.int64, device=dev)
qkv = torch.randn(B, (nq + 2 * nkv) * hd, device=dev).to(torch.bfloat16)
out = torch.empty(B, nq * hd, device=dev, dtype=torch.bfloat16)
op = {"name": "d", "kind": "Custom", "inputs": [], "outputs": [],
      "attrs": {"custom_name": "attn_decode", "params": {"heads": nq, "kv_heads": nkv, "head_dim": hd, "page_size": page,
                                                         "kv_layout": 1 if hnd else 0}}}
kvb = 2.0 * B * ctx * nkv * hd * 2
res = {}
for sms in [148, 124, 108, 92, 74, 64, 48]:
    for _ in range(3):
        of.launch(op, [qkv, kc, vc, table, pos], [out], B, max_ctas=sms)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        of.launch(op, [qkv, kc, vc, table, pos], [out], B, max_ctas=sms)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    res[sms] = round(kvb / ms / 1e6)
print(json.dumps({"lib": os.environ.get("OPF_LIB", "default"), "decode": os.environ.get("OPF_DECODE", ""),
                  "layout": "hnd" if hnd else "nhd",
                  "gbs_by_sms": res}))
