"""The drop-in boundary, exercised from the reference's side.

tests/bridge/bridge_frontend.cpp and ext_op.cu are reference-side programs:
they include the reference's headers (/root/reference/proj/include) and reach
the backend only through include/opflow_b200_bridge.hpp (the C++ adapter over
the C-ABI that rethrows opf_status as the reference's opflow::Error).

* CPU: reference GraphDescriptions from the reference's own builders, through
  the bridge, give the same graphs and plans as the reference's build_graph /
  partition, and malformed descriptions raise the same Errc through both.
* GPU: an external kernel registered with opf_register_op runs as a Custom op,
  isolated by ByFunc(custom_name), under a 2-nano-batch split, against the
  reference's eval_reference with an oracle CustomFn of the same op.
* Python: the same registry through opflow.register_op (ctypes CFUNCTYPE).
"""
import json
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
BR = ROOT / "tests" / "bridge"
REF_INCLUDE = Path("/root/reference/proj/include")


def _binary(name: str) -> Path:
    exe = BR / "_build" / name
    if REF_INCLUDE.exists():
        subprocess.run(["make", "-s", "-C", str(BR)], check=True)
    if not exe.exists():
        pytest.skip(f"{exe} not built (needs the reference headers)")
    return exe


@pytest.mark.usefixtures("built")
def test_bridge_frontend_matches_reference():
    exe = _binary("bridge_frontend")
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    cases = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    assert len(cases) >= 180
    errs = 0
    for c in cases:
        assert c["ref_error"] == c["ours_error"], c["case"]
        if c["ref_error"]:
            errs += 1
        if c["ref_graph"] is not None:
            rg, og = c["ref_graph"], c["ours_graph"]
            for k in ("graph_inputs", "weights", "graph_outputs"):
                assert rg[k] == og[k], (c["case"], k)
            assert [(o["name"], o["kind"], o["inputs"], o["outputs"], o["resource_class"]) for o in rg["ops"]] == \
                   [(o["name"], o["kind"], o["inputs"], o["outputs"], o["resource_class"]) for o in og["ops"]], c["case"]
            assert [(t["name"], t["shape"], t["producer"], t["consumers"]) for t in rg["tensors"]] == \
                   [(t["name"], t["shape"], t["producer"], t["consumers"]) for t in og["tensors"]], c["case"]
        if c["ref_plan"] is not None:
            rp, op = c["ref_plan"], c["ours_plan"]
            assert rp["subgraphs"] == op["subgraphs"], c["case"]
            assert rp["sg_edges"] == op["sg_edges"] and rp["op_to_subgraph"] == op["op_to_subgraph"], c["case"]
    assert errs == 6  # every malformed description raised, with the reference's Errc


@pytest.mark.gpu
@pytest.mark.usefixtures("built")
def test_external_op_registered_through_bridge(tmp_path, ref):
    exe = _binary("ext_op")
    rng = np.random.default_rng(11)
    R, H = 256, 256
    x = rng.uniform(-1, 1, (R, H)).astype(np.float32)
    w = (rng.uniform(-1, 1, (H, H)) * 0.3).astype(np.float32)
    (tmp_path / "in.bin").write_bytes(x.tobytes() + w.tobytes())
    r = subprocess.run([str(exe), str(tmp_path / "in.bin"), str(tmp_path / "out.bin"), str(tmp_path / "desc.json")],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-3000:]
    info = json.loads(r.stdout.strip().splitlines()[-1])
    # the plan isolates the external op (ByFunc on its custom_name), the split
    # ran it once per nano-batch (two host calls at capture, then replays)
    labels = [s["label"] for s in info["plan"]["subgraphs"]]
    assert "blk.cap" in labels and len(labels) == 3, labels
    assert info["calls"] == 2
    assert info["stats"]["last"]["dispatches"] >= 6 and info["stats"]["last"]["copied_elements"] == 0
    got = np.frombuffer((tmp_path / "out.bin").read_bytes(), dtype=np.float32).reshape(R, H)
    want = ref.evaluate((tmp_path / "desc.json").read_text(), R, {"x": x, "w": w})["y"]
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)


@pytest.mark.gpu
@pytest.mark.usefixtures("built")
def test_python_registered_op(cuda, ref):
    """opflow.register_op: a Python callable (torch kernels on the engine's
    stream, writing into the caller-owned output views) as a registered
    device op, captured into the engine's CUDA graph like a built-in."""
    import torch
    from paper_2605_21603_b200 import opflow as of
    calls = []

    def softcap(ctx, ins, outs, rows, stream):
        calls.append(rows)
        cap = ctx.params["cap"]
        with torch.cuda.stream(stream):
            torch.div(ins[0], cap, out=outs[0])
            outs[0].tanh_().mul_(cap)

    of.register_op("softcap_py", softcap, of.ResourceClass.kMemory, 1, 1)
    R, H = 256, 256
    desc = {"tensors": [{"name": "x", "shape": [R, H], "dtype": "f32", "role": "input"},
                        {"name": "w", "shape": [H, H], "batch": "replicated", "dtype": "f32", "role": "weight"},
                        {"name": "mm", "shape": [R, H], "dtype": "f32", "role": "intermediate"},
                        {"name": "capped", "shape": [R, H], "dtype": "f32", "role": "intermediate"},
                        {"name": "y", "shape": [R, H], "dtype": "f32", "role": "output"}],
            "operators": [{"name": "blk.proj", "kind": "MatMul", "inputs": ["x", "w"], "outputs": ["mm"],
                           "module_path": "blk.proj"},
                          {"name": "blk.cap", "kind": "Custom", "inputs": ["mm"], "outputs": ["capped"],
                           "module_path": "blk.cap", "attrs": {"custom_name": "softcap_py", "params": {"cap": 2.0}}},
                          {"name": "blk.norm", "kind": "RowScale", "inputs": ["capped"], "outputs": ["y"],
                           "module_path": "blk.norm"}]}
    g = of.build_graph(desc)
    plan = of.partition(g, [of.PartitionRule.by_func("softcap_py")])
    assert [s.label for s in plan.subgraphs] == ["filler#0", "blk.cap", "filler#2"]
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (R, H)).astype(np.float32)
    w = (rng.uniform(-1, 1, (H, H)) * 0.3).astype(np.float32)
    sess = of.Session(g, plan, {"lanes": 2})
    xt, wt = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    yt = torch.empty(R, H, device="cuda")
    sess.bind("x", xt), sess.bind("w", wt), sess.bind("y", yt)
    for _ in range(3):
        sess.run({"name": "split_overlap", "n_microbatches": 2, "lane_mode": "ubatch"})
    sess.check()
    assert calls == [128, 128]  # once per nano-batch at capture; replays do not call back
    want = dict(desc)
    want["operators"] = [dict(o) for o in desc["operators"]]
    want["operators"][1]["attrs"] = {"custom_name": "softcap", "params": {"cap": 2.0}}
    ref_y = ref.evaluate(json.dumps(want), R, {"x": x, "w": w})["y"]
    np.testing.assert_allclose(yt.cpu().numpy(), ref_y, rtol=1e-5, atol=1e-5)
