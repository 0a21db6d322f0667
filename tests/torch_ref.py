"""Plain PyTorch fp32 reference of the Llama / Qwen3-MoE graph descriptions,
evaluated on the GPU (test infrastructure): the full-size counterpart of the
numpy oracle (oracle/oracle.py), same op semantics, so parity can be checked
at BASELINE.json's bench shapes where the numpy oracle would take hours."""
from __future__ import annotations

import json
import math

import torch


def _rms(x, g, eps):
    return x * torch.rsqrt((x * x).mean(dim=1, keepdim=True) + eps) * g


def _rope(qkv, pos, heads, kv_heads, hd, theta):
    T = qkv.shape[0]
    h = qkv.view(T, heads + 2 * kv_heads, hd).clone()
    half = hd // 2
    inv = theta ** (-torch.arange(0, half, device=qkv.device, dtype=torch.float32) * 2.0 / hd)
    ang = pos.float()[:, None] * inv[None, :]
    c, s = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
    n = heads + kv_heads
    a, b = h[:, :n, :half].clone(), h[:, :n, half:].clone()
    h[:, :n, :half] = a * c - b * s
    h[:, :n, half:] = b * c + a * s
    return h.view(T, -1)


def _attn_prefill(qkv, heads, kv_heads, hd, S):
    T = qkv.shape[0]
    n = T // S
    x = qkv.view(n, S, heads + 2 * kv_heads, hd)
    q = x[:, :, :heads].permute(0, 2, 1, 3)
    k = x[:, :, heads:heads + kv_heads].permute(0, 2, 1, 3).repeat_interleave(heads // kv_heads, dim=1)
    v = x[:, :, heads + kv_heads:].permute(0, 2, 1, 3).repeat_interleave(heads // kv_heads, dim=1)
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
    return o.permute(0, 2, 1, 3).reshape(T, heads * hd)


def _attn_decode(qkv, kc, vc, table, ctx, heads, kv_heads, hd, page, kv_layout, chunk=16):
    B = qkv.shape[0]
    out = torch.empty(B, heads * hd, device=qkv.device, dtype=torch.float32)
    grp = heads // kv_heads
    for b0 in range(0, B, chunk):
        for b in range(b0, min(B, b0 + chunk)):
            n = int(ctx[b])
            pages = table[b, : (n + page - 1) // page]
            kk, vv = kc[pages], vc[pages]
            if kv_layout == 1:  # [p, kvh, page, hd] -> [p, page, kvh, hd]
                kk, vv = kk.transpose(1, 2), vv.transpose(1, 2)
            kk = kk.reshape(-1, kv_heads, hd)[:n].float()
            vv = vv.reshape(-1, kv_heads, hd)[:n].float()
            row = qkv[b].float().view(heads + 2 * kv_heads, hd)
            K = torch.cat([kk, row[heads:heads + kv_heads][None]], 0)          # [n+1, kvh, hd]
            V = torch.cat([vv, row[heads + kv_heads:][None]], 0)
            q = row[:heads].view(kv_heads, grp, hd)                            # [kvh, grp, hd]
            sc = torch.einsum("kgd,nkd->kgn", q, K) / math.sqrt(hd)
            p = torch.softmax(sc, dim=-1)
            out[b] = torch.einsum("kgn,nkd->kgd", p, V).reshape(-1)
    return out


def _route(ids, E):
    flat = ids.reshape(-1)
    valid = (flat >= 0) & (flat < E)
    key = torch.where(valid, flat, torch.full_like(flat, E))
    order = torch.argsort(key, stable=True)
    pos = torch.empty_like(order)
    pos[order] = torch.arange(flat.numel(), device=ids.device)
    slot = torch.where(valid, pos, torch.full_like(pos, -1)).view(ids.shape)
    return slot, key[order]


def evaluate(desc_json: str, rows: int, bind: dict) -> dict:
    """bind: name -> device tensor (any dtype); returns {output name: fp32 tensor}.
    bf16 tensors are computed in fp32, with bf16 rounding at the points the
    engine stores bf16 intermediates (every op output of a bf16 graph)."""
    d = json.loads(desc_json)
    meta = {t["name"]: t for t in d["tensors"]}
    env = {}
    for n, v in bind.items():
        env[n] = v.float() if v.dtype in (torch.bfloat16, torch.float16) else v

    def rnd(name, x):
        return x.to(torch.bfloat16).float() if meta[name].get("dtype") == "bf16" and x.is_floating_point() else x

    for o in d["operators"]:
        x = [env[n] for n in o["inputs"]]
        k = o["kind"]
        a = o.get("attrs", {})
        p = a.get("params", {})
        if k == "MatMul":
            r = [x[0] @ x[1]]
        elif k == "ElemAdd":
            r = [x[0] + x[1]]
        else:
            fn = a["custom_name"]
            if fn == "rmsnorm":
                r = [_rms(x[0], x[1], p.get("eps", 1e-5))]
            elif fn == "add_rmsnorm":
                s = x[0] + x[1]
                r = [s, _rms(rnd(o["outputs"][0], s), x[2], p.get("eps", 1e-5))]
            elif fn == "rope":
                r = [_rope(x[0], x[1], int(p["heads"]), int(p["kv_heads"]), int(p["head_dim"]),
                           p.get("theta", 10000.0))]
            elif fn == "qk_norm_rope":
                H, KV, hd = int(p["heads"]), int(p["kv_heads"]), int(p["head_dim"])
                eps = p.get("eps", 1e-6)
                T = x[0].shape[0]
                h = x[0].view(T, H + 2 * KV, hd).clone()
                for lo, hi, g in ((0, H, x[2]), (H, H + KV, x[3])):
                    seg = h[:, lo:hi]
                    h[:, lo:hi] = seg * torch.rsqrt((seg * seg).mean(-1, keepdim=True) + eps) * g
                r = [_rope(h.view(T, -1), x[1], H, KV, hd, p.get("theta", 1e6))]
            elif fn == "silu_mul":
                n = x[0].shape[1] // 2
                r = [torch.nn.functional.silu(x[0][:, :n]) * x[0][:, n:]]
            elif fn == "attn_prefill":
                r = [_attn_prefill(x[0], int(p["heads"]), int(p["kv_heads"]), int(p["head_dim"]),
                                   int(p["seq_len"]))]
            elif fn == "kv_write":
                r = [x[1]]  # the step's own attention reads only earlier positions
            elif fn == "attn_decode":
                r = [_attn_decode(x[0], bind[o["inputs"][1]], bind[o["inputs"][2]], x[3], x[4],
                                  int(p["heads"]), int(p["kv_heads"]), int(p["head_dim"]),
                                  int(p.get("page_size", 16)), int(p.get("kv_layout", 0)))]
            elif fn == "moe_topk":
                kk = int(p.get("topk", 8))
                # (value desc, index asc), like the engine and the oracle
                v, ids = torch.sort(x[0], dim=1, descending=True, stable=True)
                v, ids = v[:, :kk], ids[:, :kk]
                e = torch.exp(v - v[:, :1])
                den = e.sum(1, keepdim=True) if p.get("renorm", 1) else torch.exp(x[0] - v[:, :1]).sum(1, keepdim=True)
                r = [ids.to(torch.int64), e / den]
            elif fn == "moe_dispatch":
                E = int(p.get("experts", 128))
                T, kk = x[1].shape
                slot, _ = _route(x[1], E)
                xd = torch.zeros(T * kk, x[0].shape[1], device=x[0].device)
                s = slot.reshape(-1)
                tok = torch.arange(T, device=x[0].device).repeat_interleave(kk)
                ok = s >= 0
                xd[s[ok]] = x[0][tok[ok]]
                r = [xd.view(T, -1), slot]
            elif fn in ("moe_gate_up", "moe_down"):
                E = int(p.get("experts", 128))
                T, kk = x[1].shape
                _, rexp = _route(x[1], E)
                w = bind[o["inputs"][2]].float()
                K = w.shape[1]
                act = x[0].view(T * kk, K)
                gate_up = fn == "moe_gate_up"
                nout = w.shape[2] // 2 if gate_up else w.shape[2]
                out = torch.zeros(T * kk, nout, device=act.device)
                for e_ in range(E):
                    rows_e = torch.nonzero(rexp == e_).flatten()
                    if rows_e.numel() == 0:
                        continue
                    y = act[rows_e] @ w[e_]
                    if gate_up:
                        y = torch.nn.functional.silu(y[:, :nout]) * y[:, nout:]
                    out[rows_e] = y
                r = [out.view(T, -1)]
            elif fn == "moe_combine":
                slot, w = x[1], x[2]
                T, kk = slot.shape
                Hh = x[0].shape[1] // kk
                rws = x[0].view(T * kk, Hh)
                y = torch.zeros(T, Hh, device=rws.device)
                for j in range(kk):
                    s = slot[:, j]
                    ok = s >= 0
                    y[ok] += w[ok, j:j + 1] * rws[s[ok]]
                r = [y]
            else:
                raise KeyError(f"torch_ref: no reference for '{fn}'")
        for n, v in zip(o["outputs"], r):
            env[n] = rnd(n, v)
    return {t["name"]: env[t["name"]] for t in d["tensors"] if t["role"] == "output"}
