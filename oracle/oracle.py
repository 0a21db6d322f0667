"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference's CPU path.

This is the parity oracle, never the product: only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / reference legs may import it.

Restated algorithms (each cites the reference file:line it follows):
  * topological order: Kahn with min-declaration-index frontier
    (/root/reference/proj/src/graph.cpp:175-201)
  * eval_reference: ops in topological order (/root/reference/proj/src/eval.cpp:109-165)
  * stand-in kernels, bit-exact in fp32 / wrapping int64
    (/root/reference/proj/src/kernels_scalar.cpp:13-113):
      MatMul   i-k-j, one fp32 rounding per product and per sum
      RowScale x / sqrt(mean(x^2) + 1e-6f) (fp32, sequential sum) | x / max(1,max|x|) (i64)
      AllReduce x * world_size; AllToAll column gather; Attention row prefix sum
  * alltoall_permutation: mt19937_64 + libstdc++ std::shuffle (two-draw Lemire
    path) (/root/reference/proj/src/eval.cpp:14-20) — pinned against the
    compiled reference in tests/test_oracle.py.
Extensions (parity unpinned in the reference, which has no Llama semantics;
SURVEY.md §8c.6): rmsnorm, add_rmsnorm, rope, attn_prefill, attn_decode,
silu_mul — fp32/fp64 numpy, cross-checked against oracle/ref_shim.cpp and torch;
qk_norm_rope and the MoE ops (moe_topk / moe_route / dispatch / experts / combine),
restating the published Qwen3-MoE layer (parity unpinned, pinned here by tests).
"""
from __future__ import annotations

import heapq
import json
from typing import Dict, List, Optional

import numpy as np

MASK64 = (1 << 64) - 1


# ------------------------------------------------------------------ mt19937_64 + std::shuffle
class MT19937_64:
    N, M = 312, 156
    A = 0xB5026F5AA96619E9
    UPPER, LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int):
        self.mt = [0] * self.N
        self.mt[0] = seed & MASK64
        for i in range(1, self.N):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & MASK64
        self.idx = self.N

    def _twist(self):
        mt = self.mt
        for i in range(self.N):
            x = (mt[i] & self.UPPER) | (mt[(i + 1) % self.N] & self.LOWER)
            xa = x >> 1
            if x & 1:
                xa ^= self.A
            mt[i] = mt[(i + self.M) % self.N] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self.N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64


def _uniform(g: MT19937_64, lo: int, hi: int) -> int:
    """libstdc++ uniform_int_distribution<uint64> on a 64-bit URBG (Lemire _S_nd)."""
    rng = hi - lo + 1
    prod = g() * rng
    low = prod & MASK64
    if low < rng:
        threshold = ((-rng) & MASK64) % rng
        while low < threshold:
            prod = g() * rng
            low = prod & MASK64
    return lo + (prod >> 64)


def alltoall_permutation(seed: int, cols: int) -> List[int]:
    p = list(range(cols))
    if cols == 0:
        return p
    g = MT19937_64((seed * 0x9E3779B97F4A7C15 + cols) & MASK64)
    urange = cols
    # libstdc++ std::shuffle: pairs of swap positions from one draw when the
    # generator range covers urange^2 (always true for 64-bit and cols < 2^32)
    i = 1
    if urange % 2 == 0:
        j = _uniform(g, 0, 1)
        p[i], p[j] = p[j], p[i]
        i += 1
    while i != cols:
        swap_range = i + 1
        x = _uniform(g, 0, swap_range * (swap_range + 1) - 1)
        a, b = x // (swap_range + 1), x % (swap_range + 1)
        p[i], p[a] = p[a], p[i]
        i += 1
        p[i], p[b] = p[b], p[i]
        i += 1
    return p


# ------------------------------------------------------------------ stand-in kernels
def matmul(a: np.ndarray, w: np.ndarray, exact: bool = True) -> np.ndarray:
    if a.dtype == np.int64:
        out = np.zeros((a.shape[0], w.shape[1]), dtype=np.int64)
        with np.errstate(over="ignore"):
            for k in range(a.shape[1]):
                out += a[:, k:k + 1] * w[k:k + 1, :]
        return out
    if not exact:
        return (a.astype(np.float64) @ w.astype(np.float64)).astype(np.float32)
    out = np.zeros((a.shape[0], w.shape[1]), dtype=np.float32)
    for k in range(a.shape[1]):
        out += a[:, k:k + 1] * w[k:k + 1, :]  # fp32 multiply, then fp32 add
    return out


def row_scale(x: np.ndarray) -> np.ndarray:
    if x.dtype == np.int64:
        with np.errstate(over="ignore"):
            mag = np.where(x < 0, np.negative(x), x)
        stat = np.maximum(mag.max(axis=1, keepdims=True), 1)
        q = x // stat
        q = q + ((x < 0) & (x % stat != 0))
        return q.astype(np.int64)
    sumsq = np.zeros(x.shape[0], dtype=np.float32)
    for c in range(x.shape[1]):
        sumsq += x[:, c] * x[:, c]
    inv = np.float32(1.0) / np.sqrt(sumsq / np.float32(x.shape[1]) + np.float32(1e-6))
    return x * inv[:, None]


def prefix_sum(x: np.ndarray) -> np.ndarray:
    out = np.empty_like(x)
    acc = np.zeros(x.shape[0], dtype=x.dtype)
    with np.errstate(over="ignore"):
        for c in range(x.shape[1]):
            acc = acc + x[:, c]
            out[:, c] = acc
    return out


def scale(x: np.ndarray, f: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        if x.dtype == np.int64:
            return x * np.int64(f)
        return x * np.float32(f)


# ------------------------------------------------------------------ Llama extensions (fp32)
def rmsnorm(x, g, eps):
    x64 = x.astype(np.float64)
    inv = 1.0 / np.sqrt((x64 * x64).mean(axis=1, keepdims=True) + eps)
    return (x64 * inv * g.astype(np.float64)).astype(np.float32)


def rope(qkv, pos, heads, kv_heads, head_dim, theta):
    y = qkv.astype(np.float32).copy()
    half = head_dim // 2
    inv = theta ** (-2.0 * np.arange(half) / head_dim)
    ang = pos.astype(np.float64)[:, None] * inv[None, :]
    c, s = np.cos(ang), np.sin(ang)
    for h in range(heads + kv_heads):
        a = qkv[:, h * head_dim:h * head_dim + half].astype(np.float64)
        b = qkv[:, h * head_dim + half:(h + 1) * head_dim].astype(np.float64)
        y[:, h * head_dim:h * head_dim + half] = a * c - b * s
        y[:, h * head_dim + half:(h + 1) * head_dim] = b * c + a * s
    return y


def silu_mul(gu):
    I = gu.shape[1] // 2
    g = gu[:, :I].astype(np.float64)
    return (g / (1.0 + np.exp(-g)) * gu[:, I:]).astype(np.float32)


def round_bf16(a):
    """Round-to-nearest-even to bf16, returned as float32 (storage contract of bf16 tensors)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32)


# ------------------------------------------------------------------ Qwen3 extensions
# No Qwen3 / MoE semantics exist in the reference (SURVEY §8c gotcha 6): these
# restate the published Qwen3 layer (HF modeling_qwen3_moe: q_norm/k_norm before
# RoPE; router softmax over the selected top-k when norm_topk_prob) in fp64.
def qk_norm_rope(qkv, pos, qn, kn, heads, kv_heads, head_dim, theta, eps):
    y = qkv.astype(np.float64).copy()
    for h in range(heads + kv_heads):
        blk = y[:, h * head_dim:(h + 1) * head_dim]
        g = (qn if h < heads else kn).astype(np.float64)
        y[:, h * head_dim:(h + 1) * head_dim] = blk / np.sqrt((blk * blk).mean(axis=1, keepdims=True) + eps) * g
    return rope(y, pos, heads, kv_heads, head_dim, theta)


def moe_topk(logits, k, renorm=True):
    """ids = top-k by (value desc, index asc); w = softmax over the selected k
    logits (renorm) or the full-softmax probabilities of the selected experts."""
    l64 = logits.astype(np.float64)
    order = np.argsort(-l64, axis=1, kind="stable")
    ids = order[:, :k].astype(np.int64)
    v = np.take_along_axis(l64, ids, axis=1)
    e = np.exp(v - v[:, :1])
    denom = e.sum(axis=1, keepdims=True) if renorm else np.exp(l64 - v[:, :1]).sum(axis=1, keepdims=True)
    return ids, (e / denom).astype(np.float32)


def moe_route(ids, experts):
    """Stable counting sort of the T*k (token, j) slots by expert: slot[t, j] =
    row of (t, j) in the expert-sorted layout (-1 for ids outside [0, E)), and
    the expert of every sorted row."""
    flat = ids.reshape(-1)
    valid = (flat >= 0) & (flat < experts)
    key = np.where(valid, flat, experts)
    order = np.argsort(key, kind="stable")
    pos = np.empty(flat.size, dtype=np.int64)
    pos[order] = np.arange(flat.size)
    slot = np.where(valid, pos, -1).reshape(ids.shape)
    return slot, key[order]


def moe_dispatch(x, ids, experts):
    T, k = ids.shape
    H = x.shape[1]
    slot, _ = moe_route(ids, experts)
    xd = np.zeros((T * k, H), dtype=np.float32)
    s = slot.reshape(-1)
    tok = np.repeat(np.arange(T), k)
    ok = s >= 0
    xd[s[ok]] = x[tok[ok]]
    return xd.reshape(T, k * H), slot


def moe_experts(act, ids, w, experts, gate_up):
    """Grouped expert MatMul over the dispatched rows; w = [E, K, N] per-expert
    [K, N] weights; gate_up fuses SiLU(gate) * up (gate = columns [0, N/2))."""
    T, k = ids.shape
    _, row_expert = moe_route(ids, experts)
    K = w.shape[1]
    a = act.reshape(T * k, K).astype(np.float64)
    n_out = w.shape[2] // 2 if gate_up else w.shape[2]
    out = np.zeros((T * k, n_out), dtype=np.float32)
    for e in range(experts):
        rows = np.nonzero(row_expert == e)[0]
        if rows.size == 0:
            continue
        y = a[rows] @ w[e].astype(np.float64)
        if gate_up:
            g, u = y[:, :n_out], y[:, n_out:]
            y = g / (1.0 + np.exp(-g)) * u
        out[rows] = y
    return out.reshape(T, k * n_out)


def moe_combine(yd, slot, w):
    T, k = slot.shape
    H = yd.shape[1] // k
    rows = yd.reshape(T * k, H).astype(np.float64)
    y = np.zeros((T, H), dtype=np.float64)
    for j in range(k):
        s = slot[:, j]
        ok = s >= 0
        y[ok] += w[ok, j:j + 1].astype(np.float64) * rows[s[ok]]
    return y.astype(np.float32)


def attn_prefill(qkv, heads, kv_heads, head_dim, seq_len):
    rows = qkv.shape[0]
    out = np.zeros((rows, heads * head_dim), dtype=np.float32)
    grp = heads // kv_heads
    scale_ = 1.0 / np.sqrt(head_dim)
    mask = np.triu(np.ones((seq_len, seq_len), dtype=bool), 1)
    for s0 in range(0, rows, seq_len):
        blk = qkv[s0:s0 + seq_len].astype(np.float64)
        for h in range(heads):
            kh = h // grp
            q = blk[:, h * head_dim:(h + 1) * head_dim]
            k = blk[:, (heads + kh) * head_dim:(heads + kh + 1) * head_dim]
            v = blk[:, (heads + kv_heads + kh) * head_dim:(heads + kv_heads + kh + 1) * head_dim]
            sc = q @ k.T * scale_
            sc[mask] = -np.inf
            sc -= sc.max(axis=1, keepdims=True)
            p = np.exp(sc)
            p /= p.sum(axis=1, keepdims=True)
            out[s0:s0 + seq_len, h * head_dim:(h + 1) * head_dim] = p @ v
    return out


def attn_decode(qkv, kc, vc, table, ctx_len, heads, kv_heads, head_dim, page_size, kv_layout=0):
    """kv_layout 0: pages [page, kv_heads, head_dim] (NHD, the reference / vLLM
    layout); 1: pages [kv_heads, page, head_dim] (HND), read as NHD."""
    if kv_layout == 1:
        kc = np.ascontiguousarray(np.swapaxes(kc, 1, 2))
        vc = np.ascontiguousarray(np.swapaxes(vc, 1, 2))
    B = qkv.shape[0]
    out = np.zeros((B, heads * head_dim), dtype=np.float32)
    grp = heads // kv_heads
    scale_ = 1.0 / np.sqrt(head_dim)
    for b in range(B):
        n = int(ctx_len[b])
        pages = table[b, :(n + page_size - 1) // page_size]
        kk = kc[pages].reshape(-1, kv_heads, head_dim)[:n].astype(np.float64)
        vv = vc[pages].reshape(-1, kv_heads, head_dim)[:n].astype(np.float64)
        row = qkv[b].astype(np.float64)
        for h in range(heads):
            kh = h // grp
            q = row[h * head_dim:(h + 1) * head_dim]
            kcur = row[(heads + kh) * head_dim:(heads + kh + 1) * head_dim]
            vcur = row[(heads + kv_heads + kh) * head_dim:(heads + kv_heads + kh + 1) * head_dim]
            K = np.vstack([kk[:, kh, :], kcur[None]])
            V = np.vstack([vv[:, kh, :], vcur[None]])
            sc = K @ q * scale_
            sc -= sc.max()
            p = np.exp(sc)
            out[b, h * head_dim:(h + 1) * head_dim] = (p @ V) / p.sum()
    return out


# ------------------------------------------------------------------ graph evaluation
def topo_order(desc: dict) -> List[int]:
    """Operator declaration indices in the reference's topological order."""
    ops = desc["operators"]
    producer = {}
    for i, o in enumerate(ops):
        for t in o["outputs"]:
            producer[t] = i
    succ = [[] for _ in ops]
    indeg = [0] * len(ops)
    for i, o in enumerate(ops):
        preds = sorted({producer[t] for t in o["inputs"] if t in producer and producer[t] != i})
        for p in preds:
            succ[p].append(i)
            indeg[i] += 1
    heap = [i for i in range(len(ops)) if indeg[i] == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        i = heapq.heappop(heap)
        order.append(i)
        for s in succ[i]:
            indeg[s] -= 1
            if indeg[s] == 0:
                heapq.heappush(heap, s)
    if len(order) != len(ops):
        raise ValueError("CycleDetected")
    return order


def kv_write(qkv, slots, kc, vc, heads, kv_heads, head_dim, page_size, kv_layout=0):
    """Store each row's K / V (qkv columns of head nq + kh / nq + nkv + kh) into
    its paged-cache slot (page * page_size + offset; < 0 skipped), in place."""
    for t, s in enumerate(np.asarray(slots).reshape(-1)):
        if s < 0:
            continue
        pg, off = int(s) // page_size, int(s) % page_size
        for kh in range(kv_heads):
            k = qkv[t, (heads + kh) * head_dim:(heads + kh + 1) * head_dim]
            v = qkv[t, (heads + kv_heads + kh) * head_dim:(heads + kv_heads + kh + 1) * head_dim]
            if kv_layout == 1:
                kc[pg, kh, off], vc[pg, kh, off] = k, v
            else:
                kc[pg, off, kh], vc[pg, off, kh] = k, v
    return np.asarray(slots).reshape(-1).astype(np.int64)


def evaluate(desc_json: str, rows: int, bindings: Dict[str, np.ndarray],
             exact: bool = True, allreduce=None, caches_out: Optional[Dict[str, np.ndarray]] = None
             ) -> Dict[str, np.ndarray]:
    """eval_reference restated; bf16 graphs evaluate in fp32 (oracle precision).

    `allreduce(x, world_size)` overrides the reference's single-process
    AllReduce stand-in (x * world_size, eval.cpp:63-70) with a real collective
    (used by the tensor-parallel host tests).  kv_write ops update the oracle's
    copies of the caches in place; `caches_out` (a dict) receives them after the
    step, for multi-step decode loops."""
    desc = json.loads(desc_json) if isinstance(desc_json, str) else desc_json
    tmeta = {t["name"]: t for t in desc["tensors"]}
    vals: Dict[str, np.ndarray] = {}
    for t in desc["tensors"]:
        if t["role"] in ("input", "weight"):
            dt = np.int64 if t.get("dtype") == "i64" else np.float32
            vals[t["name"]] = np.ascontiguousarray(bindings[t["name"]], dtype=dt)
    ops = desc["operators"]
    for i in topo_order(desc):
        o = ops[i]
        a = o.get("attrs", {})
        p = a.get("params", {})
        x = [vals[n] for n in o["inputs"]]
        k = o["kind"]
        if k == "MatMul":
            r = [matmul(x[0], x[1], exact and x[0].dtype == np.float32 and
                        tmeta[o["inputs"][0]].get("dtype") != "bf16")]
        elif k == "ElemAdd":
            with np.errstate(over="ignore"):
                r = [x[0] + x[1]]
        elif k == "RowScale":
            r = [row_scale(x[0])]
        elif k == "AllReduce":
            r = [allreduce(x[0], a.get("world_size", 1)) if allreduce else
                 scale(x[0], a.get("world_size", 1))]
        elif k == "AllToAll":
            perm = alltoall_permutation(a.get("seed", 0), x[0].shape[1])
            r = [x[0][:, perm]]
        elif k == "Attention":
            r = [prefix_sum(x[0])]
        else:
            fn = a["custom_name"]
            if fn == "rmsnorm":
                r = [rmsnorm(x[0], x[1], p.get("eps", 1e-5))]
            elif fn == "add_rmsnorm":
                s = (x[0].astype(np.float64) + x[1]).astype(np.float32)
                r = [s, rmsnorm(s, x[2], p.get("eps", 1e-5))]
            elif fn == "rope":
                r = [rope(x[0], x[1], int(p["heads"]), int(p["kv_heads"]), int(p["head_dim"]),
                          p.get("theta", 10000.0))]
            elif fn == "silu_mul":
                r = [silu_mul(x[0])]
            elif fn == "attn_prefill":
                r = [attn_prefill(x[0], int(p["heads"]), int(p["kv_heads"]), int(p["head_dim"]),
                                  int(p["seq_len"]))]
            elif fn == "qk_norm_rope":
                r = [qk_norm_rope(x[0], x[1], x[2], x[3], int(p["heads"]), int(p["kv_heads"]),
                                  int(p["head_dim"]), p.get("theta", 1e6), p.get("eps", 1e-6)).astype(np.float32)]
            elif fn == "moe_topk":
                lg = round_bf16(x[0]) if tmeta[o["inputs"][0]].get("dtype") == "bf16" else x[0]
                r = list(moe_topk(lg, int(p.get("topk", 8)), bool(p.get("renorm", 1))))
            elif fn == "moe_dispatch":
                r = list(moe_dispatch(x[0], x[1], int(p.get("experts", 128))))
            elif fn in ("moe_gate_up", "moe_down"):
                r = [moe_experts(x[0], x[1], x[2], int(p.get("experts", 128)), fn == "moe_gate_up")]
            elif fn == "moe_combine":
                r = [moe_combine(x[0], x[1], x[2])]
            elif fn == "kv_write":
                r = [kv_write(x[0], x[1], x[2], x[3], int(p["heads"]), int(p["kv_heads"]), int(p["head_dim"]),
                              int(p.get("page_size", 16)), int(p.get("kv_layout", 0)))]
                if caches_out is not None:
                    caches_out[o["inputs"][2]], caches_out[o["inputs"][3]] = x[2], x[3]
            elif fn == "attn_decode":
                r = [attn_decode(x[0], x[1], x[2], x[3], x[4], int(p["heads"]), int(p["kv_heads"]),
                                 int(p["head_dim"]), int(p.get("page_size", 16)), int(p.get("kv_layout", 0)))]
            else:
                raise KeyError(f"no oracle for custom op '{fn}'")
        for n, v in zip(o["outputs"], r):
            vals[n] = v
    return {t["name"]: vals[t["name"]] for t in desc["tensors"] if t["role"] == "output"}
