"""Pin the oracle before trusting it: the numpy restatement (oracle/oracle.py)
against the reference's own golden vectors and against the compiled reference
(oracle/_ref, built from /root/reference/proj/src unmodified)."""
import json
import random

import numpy as np
import pytest

from oracle import oracle
from paper_2605_21603_b200 import opflow as of
from paper_2605_21603_b200.workloads import llama_inputs, rel_err, standin_inputs
from util import random_graph, unit_costs

pytestmark = pytest.mark.usefixtures("built")


def test_kernel_known_answers():
    # /root/reference/proj/tests/test_kernels.cpp:32-80
    a = np.array([[1, 2, -3, 4]], dtype=np.int64)
    b = np.array([[3, 4, 5, -6]], dtype=np.int64)
    assert (a + b).tolist() == [[4, 6, 2, -2]]
    assert oracle.scale(a, 2).tolist() == [[2, 4, -6, 8]]
    m = np.array([[1, 2]], dtype=np.int64)
    w = np.array([[1, 0, 2], [0, 1, 3]], dtype=np.int64)
    assert oracle.matmul(m, w).tolist() == [[1, 2, 8]]
    rs = oracle.row_scale(np.array([[2, -8, 4], [0, 0, 0]], dtype=np.int64))
    assert rs.tolist() == [[0, -1, 0], [0, 0, 0]]
    assert oracle.prefix_sum(np.array([[1, 2], [3, 4]], dtype=np.int64)).tolist() == [[1, 3], [3, 7]]
    x = np.array([[10, 20, 30]], dtype=np.int64)
    assert x[:, [2, 0, 1]].tolist() == [[30, 10, 20]]


def test_int64_wraparound_extremes():
    # test_kernels.cpp:139-152 (scale_i64 with extreme factors wraps)
    a = np.array([[2**63 - 1, -2**63, -1, 123456789012345, -987654321098765, 1, 0, 42]], dtype=np.int64)
    for f in (2**63 - 1, -2**63, -3, 1000000007):
        got = oracle.scale(a, f)
        want = [((int(v) * f + 2**63) % 2**64) - 2**63 for v in a[0]]
        assert got[0].tolist() == want


def test_alltoall_permutation_pinned(ref):
    # libstdc++ 13.3, seed=1 cols=8 -> [0 5 3 6 7 1 4 2]
    assert oracle.alltoall_permutation(1, 8) == [0, 5, 3, 6, 7, 1, 4, 2]
    assert ref.alltoall_permutation(1, 8) == [0, 5, 3, 6, 7, 1, 4, 2]
    rng = random.Random(5)
    for _ in range(60):
        seed, cols = rng.randrange(2**64), rng.randint(1, 300)
        want = ref.alltoall_permutation(seed, cols)
        assert oracle.alltoall_permutation(seed, cols) == want
        assert of.alltoall_permutation(seed, cols) == want  # the product's host perm


@pytest.mark.parametrize("builder", ["dense_tp", "moe_ep", "fuse_chain"])
@pytest.mark.parametrize("dtype", ["i64", "f32"])
def test_restatement_bit_exact_vs_reference(ref, builder, dtype):
    for layers, B, H in [(1, 4, 4), (2, 6, 8), (4, 6, 8), (2, 17, 33)]:
        desc = of.builder_json(builder, layers=layers, batch=B, hidden=H, dtype=dtype, costs=unit_costs())
        ins = standin_inputs(desc, B, seed=layers * 100 + H)
        want = ref.evaluate(desc, B, ins)
        got = oracle.evaluate(desc, B, ins)
        for k in want:
            assert got[k].dtype == want[k].dtype
            assert np.array_equal(got[k].view(np.uint8), want[k].view(np.uint8)), (builder, k)


def test_straightline_dense_tp(ref):
    # test_graph.cpp:48-77,223-245: 4 layers B=6 H=8 vs an independent evaluator
    B, H, L = 6, 8, 4
    desc = of.dense_tp_graph(L, B, H, costs=unit_costs())
    rng = np.random.default_rng(42)
    ins = {"x": rng.integers(-4, 5, (B, H)).astype(np.int64)}
    for l in range(L):
        ins[f"layer{l}.w"] = rng.integers(-4, 5, (H, H)).astype(np.int64)
    cur = ins["x"].astype(object)
    for l in range(L):
        attn = np.cumsum(cur, axis=1)
        mm = attn.dot(ins[f"layer{l}.w"].astype(object)) * 2
        stat = np.maximum(np.abs(mm).max(axis=1, keepdims=True), 1)
        cur = np.array([[int(v / s) if v >= 0 else -int(-v / s) for v, s in zip(r, [st] * H)]
                        for r, st in zip(mm, stat[:, 0])], dtype=object)
        cur = np.array([[abs(v) // s * (1 if v >= 0 else -1) for v in r] for r, s in zip(mm, stat[:, 0])],
                       dtype=object)
    out = ref.evaluate(desc, B, ins)["layer3.out"]
    assert out.tolist() == cur.astype(np.int64).tolist()
    assert oracle.evaluate(desc, B, ins)["layer3.out"].tolist() == out.tolist()


def test_batch_decomposability(ref):
    # test_graph.cpp:325-408 on the restatement: random splits of every kind
    rng = random.Random(99)
    for trial in range(20):
        B, H = rng.randint(2, 9), rng.randint(1, 6)
        dt = "f32" if trial % 3 == 0 else "i64"
        for kind in ["MatMul", "ElemAdd", "RowScale", "AllReduce", "AllToAll", "Attention"]:
            tensors = [{"name": "x", "shape": [B, H], "dtype": dt, "role": "input"}]
            op = {"name": "op", "kind": kind, "inputs": ["x"], "outputs": ["y"], "attrs": {}}
            if kind == "MatMul":
                tensors.append({"name": "w", "shape": [H, H], "batch": "replicated", "dtype": dt, "role": "weight"})
                op["inputs"] = ["x", "w"]
            if kind == "ElemAdd":
                tensors.append({"name": "x2", "shape": [B, H], "dtype": dt, "role": "input"})
                op["inputs"] = ["x", "x2"]
            if kind == "AllReduce":
                op["attrs"]["world_size"] = 3
            if kind == "AllToAll":
                op["attrs"]["seed"] = trial
            tensors.append({"name": "y", "shape": [B, H], "dtype": dt, "role": "output"})
            desc = json.dumps({"tensors": tensors, "operators": [op]})
            ins = standin_inputs(desc, B, seed=trial)
            full = oracle.evaluate(desc, B, ins)["y"]
            assert np.array_equal(full, ref.evaluate(desc, B, ins)["y"])
            parts, off = [], 0
            while off < B:
                s = rng.randint(1, B - off)
                part = {k: (v[off:off + s] if k in ("x", "x2") else v) for k, v in ins.items()}
                parts.append(oracle.evaluate(desc, s, part)["y"])
                off += s
            merged = np.concatenate(parts)
            if dt == "i64":
                assert np.array_equal(merged, full)
            else:
                np.testing.assert_allclose(merged, full, rtol=1e-6, atol=1e-9)


def test_llama_extensions_restatement_vs_reference_shim(ref):
    """The two CPU restatements of the Llama Custom ops (numpy / C++ CustomFn in
    the reference's registry) agree, end to end through eval_reference."""
    desc = of.toy_decoder_graph(layers=1, tokens=256, seq_len=128)
    ins = llama_inputs(desc, 256, seed=3)
    want = ref.evaluate(desc, 256, ins)
    got = oracle.evaluate(desc, 256, ins, exact=False)
    for k in want:
        assert rel_err(got[k], want[k]) < 1e-5


def test_llama_decode_restatement_vs_reference_shim(ref):
    desc = of.llama_decode_graph(layers=1, tokens=4, hidden=128, heads=4, kv_heads=2, head_dim=32,
                                 inter=256, ctx_len=40, page_size=16, dtype="f32")
    ins = llama_inputs(desc, 4, seed=9, ctx_len=37)
    want = ref.evaluate(desc, 4, ins)
    got = oracle.evaluate(desc, 4, ins, exact=False)
    for k in want:
        assert rel_err(got[k], want[k]) < 1e-5


def test_llama_extensions_vs_torch_fp32():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x = rng.standard_normal((64, 256)).astype(np.float32)
    g = (1 + 0.1 * rng.standard_normal(256)).astype(np.float32)
    t = torch.from_numpy(x)
    want = t * torch.rsqrt(t.pow(2).mean(-1, keepdim=True) + 1e-5) * torch.from_numpy(g)
    assert rel_err(oracle.rmsnorm(x, g, 1e-5), want.numpy()) < 1e-6
    gu = rng.standard_normal((8, 64)).astype(np.float32)
    tg = torch.from_numpy(gu)
    assert rel_err(oracle.silu_mul(gu), (torch.nn.functional.silu(tg[:, :32]) * tg[:, 32:]).numpy()) < 1e-6
    # causal GQA attention vs torch sdpa
    S, nq, nkv, hd = 32, 4, 2, 16
    qkv = rng.standard_normal((2 * S, (nq + 2 * nkv) * hd)).astype(np.float32)
    out = oracle.attn_prefill(qkv, nq, nkv, hd, S)
    tq = torch.from_numpy(qkv).view(2, S, nq + 2 * nkv, hd)
    q = tq[:, :, :nq].transpose(1, 2)
    k = tq[:, :, nq:nq + nkv].transpose(1, 2).repeat_interleave(nq // nkv, 1)
    v = tq[:, :, nq + nkv:].transpose(1, 2).repeat_interleave(nq // nkv, 1)
    ref_o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
    assert rel_err(out, ref_o.transpose(1, 2).reshape(2 * S, nq * hd).numpy()) < 1e-5
    # rope: HF rotate_half
    pos = np.arange(16) % 8
    qkv = rng.standard_normal((16, 3 * 32)).astype(np.float32)
    r = oracle.rope(qkv, pos, 1, 1, 32, 10000.0)
    inv = 1.0 / (10000 ** (torch.arange(0, 32, 2).double() / 32))
    ang = torch.from_numpy(pos).double()[:, None] * inv[None]
    emb = torch.cat([ang, ang], -1)
    qt = torch.from_numpy(qkv[:, :32]).double()
    rot = torch.cat([-qt[:, 16:], qt[:, :16]], -1)
    assert rel_err(r[:, :32], (qt * emb.cos() + rot * emb.sin()).numpy()) < 1e-6
    assert np.array_equal(r[:, 64:], qkv[:, 64:])
