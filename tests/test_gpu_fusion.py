"""GPU: compile-time epilogue fusion (bf16 MatMul -> silu_mul inside one
dispatch becomes one tcgen05 GEMM with a SiLU-mul epilogue) keeps parity."""
import numpy as np
import pytest

from oracle import oracle
from paper_2605_21603_b200 import opflow as of
from paper_2605_21603_b200.workloads import llama_inputs, rel_err
from test_gpu_parity import run_graph

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("built")]


@pytest.mark.parametrize("tokens,inter", [(512, 1024), (384, 2048), (130, 256)])
def test_gate_up_silu_epilogue(cuda, tokens, inter):
    desc = of.llama_graph(layers=1, tokens=tokens, seq_len=tokens if tokens % 128 else 128,
                          hidden=512, heads=4, kv_heads=2, head_dim=128, inter=inter, dtype="bf16")
    host = llama_inputs(desc, tokens, seed=inter)
    want = oracle.evaluate(desc, tokens, host, exact=False)
    fused, s1 = run_graph(desc, tokens, host, {"name": "sequential"}, config={"lanes": 3, "fuse": True})
    plain, s2 = run_graph(desc, tokens, host, {"name": "sequential"}, config={"lanes": 3, "fuse": False})
    names = [l["name"] for d in s1.schedule()["dispatches"] for l in d["launches"]]
    assert any(n.endswith("gate_up+layer0.act") for n in names), names
    assert not any("+" in l["name"] for d in s2.schedule()["dispatches"] for l in d["launches"])
    for k in want:
        assert rel_err(fused[k], want[k]) < 2e-2
        assert rel_err(fused[k], plain[k]) < 1e-2


@pytest.mark.parametrize("tokens,layers", [(512, 2), (130, 1), (384, 3)])
def test_residual_norm_epilogue(cuda, tokens, layers):
    """MatMul -> add_rmsnorm inside one dispatch (o_proj and down feeding the
    residual add + RMSNorm) runs as the epi-4 GEMM (x1 = x + A W and per-tile
    row sums of squares in the epilogue) plus one norm pass; ragged row counts
    (130) exercise the partial last tile.  Results match the unfused plan and
    the oracle, and are bitwise reproducible (no atomics in the statistics)."""
    desc = of.llama_graph(layers=layers, tokens=tokens, seq_len=tokens if tokens % 128 else 128,
                          hidden=512, heads=4, kv_heads=2, head_dim=128, inter=1024, dtype="bf16")
    host = llama_inputs(desc, tokens, seed=tokens + layers)
    want = oracle.evaluate(desc, tokens, host, exact=False)
    fused, s1 = run_graph(desc, tokens, host, {"name": "sequential"}, config={"lanes": 3})
    again, _ = run_graph(desc, tokens, host, {"name": "sequential"}, config={"lanes": 3})
    plain, s2 = run_graph(desc, tokens, host, {"name": "sequential"},
                          config={"lanes": 3, "fuse_addnorm": False})
    names = [l["name"] for d in s1.schedule()["dispatches"] for l in d["launches"]]
    assert any(n.endswith("o_proj+layer0.attn_resid_norm") for n in names), names
    assert not any("resid_norm" in n and "+" in n
                   for n in [l["name"] for d in s2.schedule()["dispatches"] for l in d["launches"]])
    assert s1.stats()["last"]["launches"] < s2.stats()["last"]["launches"]
    for k in want:
        assert rel_err(fused[k], want[k]) < 2e-2, k
        assert rel_err(fused[k], plain[k]) < 1e-2, k
        assert np.array_equal(fused[k], again[k]), k
