"""Per-tile timeline of the 2-CTA tcgen05 GEMM (cluster 0's leader CTA) on
one shape: producer first-stage wait, MMA accumulator wait / first full
stage / commit, epilogue tfull wait / release / done, in SM cycles.
Needs the -DOPF_GEMM_TRACE variant:
  python tools/build_variant.py kernels/gemm.cu paper_2605_21603_b200/_build/libopflow_trace.so -DOPF_GEMM_TRACE
  OPF_LIB=paper_2605_21603_b200/_build/libopflow_trace.so python tools/gemm_trace.py 8192 4096 512"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_21603_b200 import _lib, opflow as of  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
rope = len(sys.argv) > 4 and sys.argv[4] == "rope"  # MatMul -> rope (fused into the GEMM epilogue, EPI 2)
dev = torch.device("cuda:0")
tens = [{"name": "a", "shape": [m, k], "dtype": "bf16", "role": "input"},
        {"name": "w", "shape": [k, n], "batch": "replicated", "dtype": "bf16", "role": "weight"},
        {"name": "c", "shape": [m, n], "dtype": "bf16", "role": "output"}]
ops = [{"name": "mm", "kind": "MatMul", "inputs": ["a", "w"], "outputs": ["c"]}]
if rope:  # Llama GQA: n = (nq + 2 nkv) * 128 with nq = 4 nkv
    nkv = n // 128 // 6
    tens[2] = {"name": "qkv", "shape": [m, n], "dtype": "bf16"}
    tens += [{"name": "pos", "shape": [m], "dtype": "i64", "role": "input"},
             {"name": "c", "shape": [m, n], "dtype": "bf16", "role": "output"}]
    ops.append({"name": "rope", "kind": "Custom", "inputs": ["qkv", "pos"], "outputs": ["c"],
                "attrs": {"custom_name": "rope", "params": {"heads": 4 * nkv, "kv_heads": nkv, "head_dim": 128,
                                                             "theta": 500000.0}}})
    ops[0]["outputs"] = ["qkv"]
g = of.build_graph(json.dumps({"tensors": tens, "operators": ops}))
s = of.Session(g, of.partition(g, []), {"lanes": 1})
a = torch.randn(m, k, device=dev).to(torch.bfloat16)
w = (torch.randn(k, n, device=dev) / k ** 0.5).to(torch.bfloat16)
c = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
s.bind("a", a), s.bind("w", w), s.bind("c", c)
if rope:
    s.bind("pos", torch.arange(m, device=dev, dtype=torch.int64) % 1024)
L = _lib.lib()
buf = (C.c_ulonglong * (3 * 2048))()
cnt = (C.c_int * 3)()
for _ in range(20):
    s.run()
torch.cuda.synchronize()
L.opf_debug_gemm_trace(buf, cnt)  # reset
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
s.run()
e1.record()
torch.cuda.synchronize()
L.opf_debug_gemm_trace(buf, cnt)
us = e0.elapsed_time(e1) * 1e3
recs = []
for r in range(3):
    for i in range(min(cnt[r], 2048)):
        v = buf[r * 2048 + i]
        recs.append((v & 0xFFFFFFFFFF, r, v >> 56, (v >> 40) & 0xFFFF))
t0 = min(x[0] for x in recs)
names = {(0, 0): "P.tile", (0, 1): "P.stage0", (1, 0): "M.tile", (1, 1): "M.accfree", (1, 2): "M.full",
         (1, 3): "M.commit", (2, 0): "E.tile", (2, 1): "E.tfull", (2, 2): "E.release", (2, 3): "E.done", (2, 4): "E.tmemld", (2, 5): "E.stored"}
print(f"shape {m}x{n}x{k}: {us:.1f} us for the launch; cluster-0 leader timeline (cycles from first event):")
for t, r, ev, u in sorted(recs):
    print(f"{t - t0:9d}  unit {u:4d}  {names[(r, ev)]}")
