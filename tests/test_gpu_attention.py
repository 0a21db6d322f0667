"""GPU: paged decode attention variants (tensor-core, warp-SIMT, generic) and
the prefill kernels vs the fp64 oracle on edge cases (partial pages, empty
context, GQA group sizes, random block tables)."""
import numpy as np
import pytest

from oracle import oracle
from paper_2605_21603_b200 import opflow as of
from paper_2605_21603_b200.workloads import rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("built")]


@pytest.mark.parametrize("nq,nkv", [(8, 8), (8, 4), (8, 2), (16, 2), (32, 8)])
@pytest.mark.parametrize("impl", [0, 1, 2])
def test_decode_variants(cuda, nq, nkv, impl):
    import torch
    rng = np.random.default_rng(nq * 10 + nkv + impl)
    B, hd, page, max_pages = 9, 128, 16, 12
    ctx = np.array([0, 1, 15, 16, 17, 100, 191, 192, 37], dtype=np.int64)
    pages = B * max_pages
    kc = rng.uniform(-1, 1, (pages, page, nkv, hd)).astype(np.float32)
    vc = rng.uniform(-1, 1, (pages, page, nkv, hd)).astype(np.float32)
    table = rng.permutation(pages).reshape(B, max_pages).astype(np.int64)
    qkv = rng.uniform(-1, 1, (B, (nq + 2 * nkv) * hd)).astype(np.float32)
    tb = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)
    t_qkv, t_k, t_v = tb(qkv), tb(kc), tb(vc)
    want = oracle.attn_decode(t_qkv.float().cpu().numpy(), t_k.float().cpu().numpy(),
                              t_v.float().cpu().numpy(), table, ctx, nq, nkv, hd, page)
    out = torch.empty(B, nq * hd, dtype=torch.bfloat16, device="cuda")
    op = {"name": "d", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "attn_decode",
                    "params": {"heads": nq, "kv_heads": nkv, "head_dim": hd, "page_size": page, "impl": impl}}}
    of.launch(op, [t_qkv, t_k, t_v, torch.from_numpy(table).cuda(), torch.from_numpy(ctx).cuda()], [out], B)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for b in range(B):
        assert rel_err(got[b], want[b]) < 1e-2, (b, ctx[b], rel_err(got[b], want[b]))


def _prefill(t, nq, nkv, S, rows, max_ctas=0, offset=0, **extra):
    import torch
    op = {"name": "a", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "attn_prefill",
                    "params": dict({"heads": nq, "kv_heads": nkv, "head_dim": 128, "seq_len": S}, **extra)}}
    # offset > 0: the output is a view `offset` elements into a larger buffer
    buf = torch.empty(rows * nq * 128 + offset, dtype=torch.bfloat16, device="cuda")
    out = buf[offset:].view(rows, nq * 128)
    of.launch(op, [t], [out], rows, max_ctas=max_ctas)
    torch.cuda.synchronize()
    return out.float().cpu().numpy()


@pytest.mark.parametrize("S,nq,nkv,seqs,ramp", [
    (128, 2, 2, 1, 0.0), (256, 4, 1, 3, 0.0), (1024, 8, 2, 2, 0.0), (512, 4, 4, 2, 6.0),
    (2048, 2, 1, 1, 3.0), (384, 6, 2, 5, 0.0)])
def test_prefill_tcgen05_vs_oracle(cuda, S, nq, nkv, seqs, ramp):
    """tcgen05/TMEM prefill (impl 0) vs the fp64 oracle and the mma.sync FA2
    kernel (impl 1).  `ramp` grows |q|,|k| along the sequence so later key tiles
    raise the row max by more than the lazy-rescale threshold (exercises the
    TMEM O rescale); persistent CTAs see several items each (seqs x heads x tiles
    > 148 for the larger cases)."""
    import torch
    rng = np.random.default_rng(S * 7 + nq + seqs)
    hd, rows = 128, S * seqs
    qkv = rng.uniform(-1, 1, (rows, (nq + 2 * nkv) * hd)).astype(np.float32)
    if ramp:
        pos = (np.arange(rows) % S) / S
        qkv[:, :(nq + nkv) * hd] *= (1.0 + ramp * pos)[:, None]
    t = torch.from_numpy(qkv).cuda().to(torch.bfloat16)
    want = oracle.attn_prefill(t.float().cpu().numpy(), nq, nkv, hd, S)
    got = _prefill(t, nq, nkv, S, rows)
    fa2 = _prefill(t, nq, nkv, S, rows, impl=1)
    assert np.isfinite(got).all()
    assert rel_err(got, want) < 1e-2
    assert rel_err(fa2, want) < 1e-2
    # a 7-CTA budget: more head-pair items than CTAs, so even GQA groups take
    # the two-head kernel (few items per SM pick one head per item), every CTA
    # walking several items; and a 16-byte (not 32-byte) aligned output view
    for got2 in (_prefill(t, nq, nkv, S, rows, max_ctas=7), _prefill(t, nq, nkv, S, rows, max_ctas=7, offset=8)):
        assert rel_err(got2, want) < 1e-2
        row_err2 = np.abs(got2 - want).max(axis=1) / (np.abs(want).max(axis=1) + 1e-6)
        assert row_err2.max() < 5e-2, int(row_err2.argmax())
    # per-row check too (a wrong tile hides in a normwise error)
    row_err = np.abs(got - want).max(axis=1) / (np.abs(want).max(axis=1) + 1e-6)
    assert row_err.max() < 5e-2, int(row_err.argmax())


def test_prefill_tcgen05_capped_ctas(cuda):
    """SM-budgeted launch (max_ctas, NanoFlow lane budgets) keeps results."""
    import torch
    rng = np.random.default_rng(5)
    S, nq, nkv, seqs = 512, 4, 2, 2
    qkv = rng.uniform(-1, 1, (S * seqs, (nq + 2 * nkv) * 128)).astype(np.float32)
    t = torch.from_numpy(qkv).cuda().to(torch.bfloat16)
    want = oracle.attn_prefill(t.float().cpu().numpy(), nq, nkv, 128, S)
    op = {"name": "a", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "attn_prefill", "params": {"heads": nq, "kv_heads": nkv, "head_dim": 128, "seq_len": S}}}
    for cap in (1, 3, 17):
        out = torch.empty(S * seqs, nq * 128, dtype=torch.bfloat16, device="cuda")
        of.launch(op, [t], [out], S * seqs, max_ctas=cap)
        torch.cuda.synchronize()
        assert rel_err(out.float().cpu().numpy(), want) < 1e-2, cap


@pytest.mark.parametrize("max_ctas", [1, 3, 148])
def test_decode_tma_ring_wraps_across_items(cuda, max_ctas):
    """TMA-ring decode: a CTA streams many (sequence, kv head) items through one
    23-slot ring (wrapping many times, items of 0..45 pages, empty contexts),
    merging each item while the producer prefetches the next."""
    import torch
    rng = np.random.default_rng(max_ctas)
    B, nq, nkv, hd, page, max_pages = 40, 32, 8, 128, 16, 45
    ctx = rng.integers(0, max_pages * page, size=B).astype(np.int64)
    ctx[:3] = [0, 1, max_pages * page]
    pages = B * max_pages
    kc = rng.uniform(-1, 1, (pages, page, nkv, hd)).astype(np.float32)
    vc = rng.uniform(-1, 1, (pages, page, nkv, hd)).astype(np.float32)
    table = rng.permutation(pages).reshape(B, max_pages).astype(np.int64)
    qkv = rng.uniform(-1, 1, (B, (nq + 2 * nkv) * hd)).astype(np.float32)
    tb = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)
    t_qkv, t_k, t_v = tb(qkv), tb(kc), tb(vc)
    want = oracle.attn_decode(t_qkv.float().cpu().numpy(), t_k.float().cpu().numpy(),
                              t_v.float().cpu().numpy(), table, ctx, nq, nkv, hd, page)
    out = torch.empty(B, nq * hd, dtype=torch.bfloat16, device="cuda")
    op = {"name": "d", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "attn_decode",
                    "params": {"heads": nq, "kv_heads": nkv, "head_dim": hd, "page_size": page}}}
    of.launch(op, [t_qkv, t_k, t_v, torch.from_numpy(table).cuda(), torch.from_numpy(ctx).cuda()], [out], B,
              max_ctas=max_ctas)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for b in range(B):
        assert rel_err(got[b], want[b]) < 1e-2, (b, ctx[b], rel_err(got[b], want[b]))


@pytest.mark.parametrize("nq,nkv", [(32, 8), (8, 2), (16, 16)])
def test_decode_hnd_layout_matches_nhd(cuda, nq, nkv):
    """kv_layout 1 (HND pages [kv_heads, page, hd]) gives the same attention as
    the reference NHD layout on the same cache contents (transposed), and both
    match the oracle."""
    import torch
    rng = np.random.default_rng(nq + nkv)
    B, hd, page, max_pages = 11, 128, 16, 20
    ctx = rng.integers(0, max_pages * page, size=B).astype(np.int64)
    ctx[:2] = [0, max_pages * page]
    pages = B * max_pages
    kc = rng.uniform(-1, 1, (pages, page, nkv, hd)).astype(np.float32)
    vc = rng.uniform(-1, 1, (pages, page, nkv, hd)).astype(np.float32)
    table = rng.permutation(pages).reshape(B, max_pages).astype(np.int64)
    qkv = rng.uniform(-1, 1, (B, (nq + 2 * nkv) * hd)).astype(np.float32)
    tb = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.bfloat16)
    t_qkv, t_k, t_v = tb(qkv), tb(kc), tb(vc)
    t_kh, t_vh = t_k.transpose(1, 2).contiguous(), t_v.transpose(1, 2).contiguous()
    want = oracle.attn_decode(t_qkv.float().cpu().numpy(), t_kh.float().cpu().numpy(), t_vh.float().cpu().numpy(),
                              table, ctx, nq, nkv, hd, page, kv_layout=1)
    outs = []
    for lay, (k, v) in [(0, (t_k, t_v)), (1, (t_kh, t_vh))]:
        out = torch.empty(B, nq * hd, dtype=torch.bfloat16, device="cuda")
        op = {"name": "d", "kind": "Custom", "inputs": [], "outputs": [],
              "attrs": {"custom_name": "attn_decode",
                        "params": {"heads": nq, "kv_heads": nkv, "head_dim": hd, "page_size": page, "kv_layout": lay}}}
        of.launch(op, [t_qkv, k, v, torch.from_numpy(table).cuda(), torch.from_numpy(ctx).cuda()], [out], B)
        torch.cuda.synchronize()
        outs.append(out.float().cpu().numpy())
    assert np.array_equal(outs[0], outs[1])  # same math, same order: bit-identical
    for b in range(B):
        assert rel_err(outs[1][b], want[b]) < 1e-2


@pytest.mark.parametrize("S,nq,nkv,seqs", [(384, 6, 2, 5), (1024, 8, 2, 2), (512, 12, 4, 3)])
def test_prefill_budget_sweep_rows(cuda, S, nq, nkv, seqs):
    """Both tcgen05 prefill kernels (odd group -> one head per item, even ->
    head pairs, small budgets -> several items per CTA) over a sweep of CTA
    budgets, every output row against the oracle: a softmax warp running a tile
    ahead of its neighbours once completed the wrong P buffer's phase (whole
    32-row quarters wrong), visible under changed timing (tools/attn_stress.py)."""
    import torch
    rng = np.random.default_rng(S + nq)
    rows = S * seqs
    qkv = rng.uniform(-1, 1, (rows, (nq + 2 * nkv) * 128)).astype(np.float32)
    t = torch.from_numpy(qkv).cuda().to(torch.bfloat16)
    want = oracle.attn_prefill(t.float().cpu().numpy(), nq, nkv, 128, S)
    for cap in (1, 2, 3, 5, 7, 16, 0):
        for _ in range(3):
            got = _prefill(t, nq, nkv, S, rows, max_ctas=cap)
            row_err = np.abs(got - want).max(axis=1) / (np.abs(want).max(axis=1) + 1e-6)
            assert row_err.max() < 5e-2, (cap, int(row_err.argmax()), float(row_err.max()))


@pytest.mark.parametrize("S,nq,nkv,hd,seqs", [
    (128, 8, 8, 64, 8),    # C1 toy shape (BASELINE configs[0]); 8 row slices per (sequence, head)
    (128, 8, 2, 64, 3),    # GQA group 4
    (64, 4, 1, 128, 5),    # S <= 64 form, hd 128
    (256, 2, 2, 32, 2),    # S = 256 form, few units (16 slices)
    (37, 3, 1, 48, 4),     # S and hd not multiples of 32 (partial lanes / key columns)
    (1, 2, 1, 64, 6),      # one-token sequences
    (512, 2, 1, 64, 2),    # beyond the shared-memory form: the online SIMT kernel
])
def test_prefill_fp32_vs_oracle(cuda, S, nq, nkv, hd, seqs):
    """fp32 prefill (the C1 toy's path): the shared-memory short-sequence
    kernel for S <= 256 and the online SIMT kernel beyond, vs the fp64 oracle
    within the fp32 tolerance (rel <= 1e-4, BASELINE north_star); also a
    nano-batch row slice (a whole number of sequences) of the same input."""
    import torch
    rng = np.random.default_rng(S * 13 + nq * 3 + hd)
    rows = S * seqs
    qkv = rng.uniform(-1, 1, (rows, (nq + 2 * nkv) * hd)).astype(np.float32)
    want = oracle.attn_prefill(qkv.astype(np.float64), nq, nkv, hd, S)
    op = {"name": "a", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "attn_prefill",
                    "params": {"heads": nq, "kv_heads": nkv, "head_dim": hd, "seq_len": S}}}
    t = torch.from_numpy(qkv).cuda()
    out = torch.full((rows, nq * hd), float("nan"), dtype=torch.float32, device="cuda")
    of.launch(op, [t], [out], rows)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.isfinite(got).all()
    assert rel_err(got, want) < 1e-4, rel_err(got, want)
    row_err = np.abs(got - want).max(axis=1) / (np.abs(want).max(axis=1) + 1e-6)
    assert row_err.max() < 1e-3, int(row_err.argmax())
    if seqs > 1:  # rows of the later sequences only (an offset view, as a nano-batch)
        lo = S * (seqs // 2)
        out2 = torch.full((rows - lo, nq * hd), float("nan"), dtype=torch.float32, device="cuda")
        of.launch(op, [t[lo:]], [out2], rows - lo)
        torch.cuda.synchronize()
        assert rel_err(out2.cpu().numpy(), want[lo:]) < 1e-4
