"""A/B timing of the tcgen05 GEMM on decode / TP-sharded shapes through a
one-op Session (engine workspace, so split-K is available).  Run it twice
with different OPF_GEMM_* env settings in the same gpurun call.
Prints one JSON line {shape: us}."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_21603_b200 import _lib, opflow as of  # noqa: E402

SHAPES = [(512, 6144, 4096), (512, 4096, 4096), (512, 28672, 4096), (512, 4096, 14336),
          (256, 6144, 4096), (256, 4096, 4096), (256, 28672, 4096), (256, 4096, 14336),
          (8192, 768, 4096), (8192, 4096, 512), (8192, 3584, 4096), (8192, 4096, 1792),
          (8192, 6144, 4096), (8192, 4096, 4096), (8192, 28672, 4096), (8192, 4096, 14336)]
dev = torch.device("cuda:0")
import bench  # noqa: E402
if os.environ.get("AB_SHAPES"):
    SHAPES = [tuple(int(v) if v.isdigit() else v for v in x.split("x")) for x in os.environ["AB_SHAPES"].split(",")]
out = {}
stream = torch.cuda.current_stream(dev)


def rope_reps_ms(m, n, k, nkv, a, w, c, reps=8):
    tens, ops, binds = [], [], []
    pos = torch.arange(m, device=dev, dtype=torch.int64) % 1024
    tens.append({"name": "pos", "shape": [m], "dtype": "i64", "role": "input"})
    binds.append(("pos", pos))
    for r in range(reps):
        tens += [{"name": f"a{r}", "shape": [m, k], "dtype": "bf16", "role": "input"},
                 {"name": f"w{r}", "shape": [k, n], "dtype": "bf16", "role": "weight", "batch": "replicated"},
                 {"name": f"q{r}", "shape": [m, n], "dtype": "bf16"},
                 {"name": f"c{r}", "shape": [m, n], "dtype": "bf16", "role": "output"}]
        ops += [{"name": f"mm{r}", "kind": "MatMul", "inputs": [f"a{r}", f"w{r}"], "outputs": [f"q{r}"]},
                {"name": f"rope{r}", "kind": "Custom", "inputs": [f"q{r}", "pos"], "outputs": [f"c{r}"],
                 "attrs": {"custom_name": "rope", "params": {"heads": 4 * nkv, "kv_heads": nkv, "head_dim": 128,
                                                              "theta": 500000.0}}}]
        binds += [(f"a{r}", a if r == 0 else a.clone()), (f"w{r}", w if r == 0 else w.clone()),
                  (f"c{r}", c if r == 0 else c.clone())]
    g = of.build_graph(json.dumps({"tensors": tens, "operators": ops}))
    sess = of.Session(g, of.partition(g, []), {"lanes": 1})
    for nm, x in binds:
        sess.bind(nm, x)
    for _ in range(3):
        sess.run(None, stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        e0.record(stream)
        sess.run(None, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    del sess
    return sorted(ts)[1]
for shp in SHAPES:
    m, n, k = shp[:3]
    rope = len(shp) > 3 and shp[3] == "rope"
    # device time: 8 launches back to back in one CUDA graph, rotated A / W / C
    a = torch.randn(m, k, device=dev).to(torch.bfloat16)
    w = (torch.randn(k, n, device=dev) / k ** 0.5).to(torch.bfloat16)
    c = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    if rope:  # MatMul + rope: the engine fuses the rotation into the GEMM epilogue (EPI 2)
        nkv = n // 128 // 6
        ms = rope_reps_ms(m, n, k, nkv, a, w, c)
    else:
        op = {"name": "mm", "kind": "MatMul", "inputs": ["a", "w"], "outputs": ["c"]}
        ms = bench.graph_reps_ms(of, torch, dev, stream, [("a", a, "input"), ("w", w, "weight"), ("c", c, "output")],
                                 op, shared=(), reps=8)
    us = ms * 1e3
    out[f"{m}x{n}x{k}" + ("xrope" if rope else "")] = [round(us, 1), _lib.lib().opf_gemm_splits(m, n, k, 0),
                           round(2.0 * m * n * k / us / 1e6, 1)]
print(json.dumps({"lib": os.environ.get("OPF_LIB", "default"),
                  "env": {k: v for k, v in os.environ.items() if k.startswith("OPF_GEMM")}, "us_splits_tflops": out}))
