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
