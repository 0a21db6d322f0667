"""Synthetic workloads (seeded) for the Llama-shaped graphs and the reference
stand-in graphs, shared by tests, smoke() and bench.py.

Inputs follow SURVEY.md §8d: x ~ U(-1,1), projection weights ~ U(-1,1)/sqrt(K),
norm gains ~ 1 + U(-0.1,0.1), positions = row % seq_len (prefill) or the cached
context length (decode), block tables a seeded random page permutation.  For
bf16 graphs every float value is rounded to bf16 first, so the fp32 oracle and
the device see identical inputs.
"""
from __future__ import annotations

import json
from typing import Dict

import numpy as np


def round_bf16(a: np.ndarray) -> np.ndarray:
    """fp32 -> nearest-even bf16, returned as fp32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def rel_err(got: np.ndarray, want: np.ndarray) -> float:
    """Normwise relative error ||got - want|| / ||want|| (the tolerance metric)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (den if den > 0 else 1.0))


def _param(desc: dict, custom: str, key: str, default):
    for o in desc["operators"]:
        a = o.get("attrs", {})
        if a.get("custom_name") == custom and key in a.get("params", {}):
            return a["params"][key]
    return default


def llama_inputs(desc_json, rows: int, seed: int = 0, ctx_len: int | None = None) -> Dict[str, np.ndarray]:
    """Host arrays for every GraphInput / Weight of a llama / toy / decode graph."""
    desc = json.loads(desc_json) if isinstance(desc_json, str) else desc_json
    rng = np.random.default_rng(seed)
    bf16 = any(t.get("dtype") == "bf16" for t in desc["tensors"])
    rnd = round_bf16 if bf16 else (lambda a: np.asarray(a, dtype=np.float32))
    out: Dict[str, np.ndarray] = {}
    seq_len = int(_param(desc, "attn_prefill", "seq_len", rows))
    page = int(_param(desc, "attn_decode", "page_size", 16))
    decode = any(o.get("attrs", {}).get("custom_name") == "attn_decode" for o in desc["operators"])
    table_shape = None
    for t in desc["tensors"]:
        if t["name"] == "block_table":
            table_shape = t["shape"]
    for t in desc["tensors"]:
        name, shape, role = t["name"], list(t["shape"]), t["role"]
        if role not in ("input", "weight"):
            continue
        if t.get("batch", "batched") == "batched":
            shape[0] = rows
        if name == "positions":
            if decode:
                max_ctx = (table_shape[1] * page) if table_shape else 4096
                n = ctx_len if ctx_len is not None else max_ctx
                out[name] = np.full(rows, min(n, max_ctx), dtype=np.int64)
            else:
                out[name] = (np.arange(rows) % seq_len).astype(np.int64)
        elif name == "block_table":
            max_pages = shape[1]
            perm = rng.permutation(rows * max_pages)
            out[name] = perm.reshape(rows, max_pages).astype(np.int64)
        elif name.endswith("_cache"):
            out[name] = rnd(rng.uniform(-1.0, 1.0, size=shape).astype(np.float32))
        elif name.endswith("norm.w"):
            out[name] = rnd(1.0 + rng.uniform(-0.1, 0.1, size=shape).astype(np.float32))
        elif role == "weight":
            k = shape[-2] if len(shape) == 3 else shape[0]  # [E, K, N] expert weights
            out[name] = rnd((rng.uniform(-1.0, 1.0, size=shape) / np.sqrt(k)).astype(np.float32))
        elif t.get("dtype") == "i64":
            out[name] = rng.integers(-4, 5, size=shape).astype(np.int64)
        else:
            out[name] = rnd(rng.uniform(-1.0, 1.0, size=shape).astype(np.float32))
    return out


def standin_inputs(desc_json, rows: int, seed: int = 0) -> Dict[str, np.ndarray]:
    """Reference test_util-style bindings: i64 in [-4,4], f32 in [-1,1]."""
    desc = json.loads(desc_json) if isinstance(desc_json, str) else desc_json
    rng = np.random.default_rng(seed)
    out = {}
    for t in desc["tensors"]:
        if t["role"] not in ("input", "weight"):
            continue
        shape = list(t["shape"])
        if t.get("batch", "batched") == "batched":
            shape[0] = rows
        if t.get("dtype") == "i64":
            out[t["name"]] = rng.integers(-4, 5, size=shape).astype(np.int64)
        else:
            out[t["name"]] = rng.uniform(-1.0, 1.0, size=shape).astype(np.float32)
    return out


def shard_llama_weights(full: Dict[str, np.ndarray], rank: int, world: int, heads: int,
                        kv_heads: int, head_dim: int, inter: int) -> Dict[str, np.ndarray]:
    """Megatron-style tensor-parallel shard of tp=1 Llama weights for `rank`:
    QKV and gate_up column-parallel (this rank's q / k / v heads, gate / up
    columns), O and down row-parallel; norms replicated.  The per-rank graph is
    llama_graph(tp=world): the partial O / down outputs are summed by the
    AllReduce the builder inserts."""
    nq, nkv, I = heads // world, kv_heads // world, inter // world
    hd = head_dim
    out = {}
    for name, w in full.items():
        if name.endswith(".qkv.w"):
            q = w[:, rank * nq * hd:(rank + 1) * nq * hd]
            k0 = heads * hd
            k = w[:, k0 + rank * nkv * hd:k0 + (rank + 1) * nkv * hd]
            v0 = (heads + kv_heads) * hd
            v = w[:, v0 + rank * nkv * hd:v0 + (rank + 1) * nkv * hd]
            out[name] = np.ascontiguousarray(np.concatenate([q, k, v], axis=1))
        elif name.endswith(".o.w"):
            out[name] = np.ascontiguousarray(w[rank * nq * hd:(rank + 1) * nq * hd])
        elif name.endswith(".gate_up.w"):
            g = w[:, rank * I:(rank + 1) * I]
            u = w[:, inter + rank * I:inter + (rank + 1) * I]
            out[name] = np.ascontiguousarray(np.concatenate([g, u], axis=1))
        elif name.endswith(".down.w"):
            out[name] = np.ascontiguousarray(w[rank * I:(rank + 1) * I])
        else:
            out[name] = w
    return out
