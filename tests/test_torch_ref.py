"""The full-size GPU parity tests use a PyTorch fp32 reference of the graphs
(tests/torch_ref.py); here (CPU, small shapes) it is pinned to the numpy
oracle on the same inputs, op by op semantics included."""
import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2605_21603_b200 import opflow as of
from paper_2605_21603_b200.workloads import llama_inputs, rel_err
from torch_ref import evaluate


def _cmp(desc, rows, host, tol=1e-4):
    want = oracle.evaluate(desc, rows, host, exact=False)
    bind = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in host.items()}
    got = evaluate(desc, rows, bind)
    for k in want:
        assert rel_err(got[k].numpy(), want[k]) < tol, (k, rel_err(got[k].numpy(), want[k]))


def test_torch_ref_llama_prefill_matches_oracle():
    desc = of.llama_graph(layers=2, tokens=256, seq_len=128, hidden=256, heads=4, kv_heads=2, head_dim=128,
                          inter=512, dtype="f32")
    _cmp(desc, 256, llama_inputs(desc, 256, seed=21))


@pytest.mark.parametrize("kv_layout", [0, 1])
def test_torch_ref_llama_decode_matches_oracle(kv_layout):
    desc = of.llama_decode_graph(layers=1, tokens=6, hidden=256, heads=4, kv_heads=2, head_dim=128, inter=512,
                                 ctx_len=70, page_size=16, dtype="f32", kv_layout=kv_layout)
    _cmp(desc, 6, llama_inputs(desc, 6, seed=22, ctx_len=53))


def test_torch_ref_qwen3_moe_matches_oracle():
    desc = of.qwen3_moe_graph(layers=1, tokens=128, seq_len=64, hidden=256, heads=4, kv_heads=2, head_dim=128,
                              experts=16, topk=4, moe_inter=128, dtype="f32", ep=1)
    _cmp(desc, 128, llama_inputs(desc, 128, seed=23), tol=1e-3)
