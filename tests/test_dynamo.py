"""TorchDynamo frontend on CPU: the lowering of a plain PyTorch Llama model into
the reference's GraphDescription, its partition annotations (SplitModule /
SplitFunc / mark), and the lowered graph's semantics against the numpy oracle
(the eager model and oracle.evaluate of the lowered description agree)."""
import json

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2605_21603_b200 import dynamo as dyn
from paper_2605_21603_b200 import opflow as of
from torch_llama import Attention, Llama, init_

T, S = 256, 128


def _compile_dry(model, rules=(), x=None, pos=None):
    be = dyn.backend(rules=rules, dry=True)
    torch._dynamo.reset()
    fn = torch.compile(model, backend=be, fullgraph=True, dynamic=False)
    x = torch.rand(T, 512) * 2 - 1 if x is None else x
    pos = (torch.arange(T) % S).to(torch.int64) if pos is None else pos
    y = fn(x, pos)
    assert len(be.lowered) == 1
    return be.lowered[0], x, pos, y


def test_lowering_matches_builder_structure():
    """The compiled model lowers to the same operator sequence as the engine's
    own Llama builder (rmsnorm, MatMul, rope, attention, MatMul, add_rmsnorm,
    MatMul, silu_mul, MatMul, ElemAdd per layer), with the residual add + norm
    folded into add_rmsnorm."""
    model = init_(Llama(layers=2))
    low, *_ = _compile_dry(model)
    got = [(o["kind"], o.get("attrs", {}).get("custom_name", "")) for o in low.description["operators"]]
    ref = json.loads(of.llama_graph(layers=2, tokens=T, seq_len=S, hidden=512, heads=4, kv_heads=2, head_dim=128,
                                    inter=1024, dtype="f32"))
    want = [(o["kind"], o.get("attrs", {}).get("custom_name", "")) for o in ref["operators"]]
    # layer boundary: our graph keeps layer l's final add as the next layer's
    # add_rmsnorm input (the builder adds then re-norms in the same way)
    assert [k for k in got if k[0] == "MatMul"] == [k for k in want if k[0] == "MatMul"]
    assert sum(1 for k in got if k[1] == "attn_prefill") == 2
    assert sum(1 for k in got if k[1] == "add_rmsnorm") == 3  # attn resid x2 + layer-1 input norm
    assert sum(1 for k in got if k[0] == "ElemAdd") == 1      # the model's last residual add
    g = of.build_graph(low.json())
    assert len(g.ops) == len(got)
    weights = [t for t in low.description["tensors"] if t["role"] == "weight"]
    assert {w["name"] for w in weights} >= {"layers.0.attn.qkv.weight", "layers.1.mlp.down.weight"}
    qkv_w = [w for w in weights if w["name"] == "layers.0.attn.qkv.weight"][0]
    assert qkv_w["shape"] == [512, (4 + 4) * 128]  # bound transposed: [K, N]


def test_annotations_become_partition_rules():
    model = init_(Llama(layers=2))
    low, *_ = _compile_dry(model, rules=[dyn.SplitModule(Attention), dyn.SplitFunc("silu_mul"), "ffn0", "ffn1"])
    g = of.build_graph(low.json())
    plan = of.partition(g, low.rules)
    of.validate_plan(plan, g)
    labels = [sg.label for sg in plan.subgraphs]
    assert "layers.0.attn" in labels and "layers.1.attn" in labels
    assert sum(1 for l in labels if "ffn" in l) == 2, labels
    assert sum(1 for l in labels if ".silu_mul" in l) == 2, labels
    # a strategy plans over it without a GPU
    sched, stats = of.dry_run(g, plan, {"name": "split_overlap", "n_microbatches": 2, "align": S,
                                        "lane_mode": "ubatch"}, rows=T)
    assert stats["last"]["dispatches"] > 0 and stats["last"]["end_live_tensors"] == 0


def test_lowered_graph_semantics_match_the_eager_model():
    """oracle.evaluate(lowered description, same weights) == the eager fp32 model."""
    model = init_(Llama(layers=2), seed=3)
    low, x, pos, y = _compile_dry(model)
    params = dict(model.named_parameters())
    binds = {}
    for name, i, kind in low.inputs:
        if kind == "batched":
            binds[name] = (x if name == "x" else pos).numpy()
        else:
            p = params[name].detach()
            binds[name] = (p.t() if kind == "weight_t" else p).contiguous().numpy()
    out = oracle.evaluate(low.json(), T, binds, exact=False)
    (oname, _, _), = low.outputs
    got = out[oname]
    want = y.detach().numpy()
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 1e-4, err


def test_unsupported_op_raises_config_error():
    class Bad(torch.nn.Module):
        def forward(self, x):
            return torch.tanh(x) + x
    be = dyn.backend(dry=True)
    torch._dynamo.reset()
    fn = torch.compile(Bad(), backend=be, fullgraph=True, dynamic=False)
    with pytest.raises(Exception) as e:
        fn(torch.rand(8, 16))
    assert "unsupported op" in str(e.value)


def test_cuda_only_runtime():
    """Without dry mode the backend never runs CPU tensors (no eager fallback)."""
    model = init_(Llama(layers=1))
    be = dyn.backend()
    torch._dynamo.reset()
    fn = torch.compile(model, backend=be, fullgraph=True, dynamic=False)
    with pytest.raises(Exception) as e:
        fn(torch.rand(T, 512), (torch.arange(T) % S).to(torch.int64))
    assert "CUDA" in str(e.value)
