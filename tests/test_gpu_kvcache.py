"""GPU: the paged KV-cache path end to end — the manager hands out slots,
kv_write stores the prompt's K / V into the pages, attn_decode of the next
token over the manager's block table equals the causal prefill attention's
last row over prompt + token (fp64 oracle), in both page layouts."""
import numpy as np
import pytest

from oracle import oracle
from paper_2605_21603_b200 import opflow as of
from paper_2605_21603_b200.workloads import rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("built")]


@pytest.mark.parametrize("kv_layout", [0, 1])
@pytest.mark.parametrize("nq,nkv", [(8, 2), (32, 8)])
def test_prefill_write_then_decode_matches_causal_attention(cuda, kv_layout, nq, nkv):
    import torch
    hd, page = 128, 16
    lens = [1, 5, 16, 17, 100, 257]
    B = len(lens)
    rng = np.random.default_rng(nq + kv_layout)
    kv = of.KvCache(layers=1, pages=64, kv_heads=nkv, head_dim=hd, page_size=page, kv_layout=kv_layout)
    kc, vc = kv.cache(0, "k"), kv.cache(0, "v")
    kc.zero_(), vc.zero_()
    W = (nq + 2 * nkv) * hd
    seqs = [rng.uniform(-1, 1, (L + 1, W)).astype(np.float32) for L in lens]
    tb = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.bfloat16)
    prm = {"heads": nq, "kv_heads": nkv, "head_dim": hd, "page_size": page, "kv_layout": kv_layout}
    # prefill: the prompt tokens of every sequence, one kv_write over the concatenation
    slots, pos = kv.append(list(range(B)), lens)
    prompt = tb(np.concatenate([s[:-1] for s in seqs]))
    written = torch.empty(int(sum(lens)), dtype=torch.int64, device="cuda")
    wop = {"name": "w", "kind": "Custom", "inputs": [], "outputs": [],
           "attrs": {"custom_name": "kv_write", "params": prm}}
    of.launch(wop, [prompt, torch.from_numpy(slots).cuda(), kc, vc], [written], prompt.shape[0])
    # padding rows (slot -1) leave the cache untouched
    of.launch(wop, [tb(rng.uniform(-1, 1, (3, W))), torch.full((3,), -1, dtype=torch.int64, device="cuda"), kc, vc],
              [torch.empty(3, dtype=torch.int64, device="cuda")], 3)
    torch.cuda.synchronize()
    assert written.cpu().numpy().tolist() == slots.tolist()
    # decode: the next token of every sequence over the manager's block table
    max_pages = 20
    table, ctx = kv.block_table(list(range(B)), max_pages)
    table = np.where(table < 0, 0, table)
    cur = tb(np.stack([s[-1] for s in seqs]))
    out = torch.empty(B, nq * hd, dtype=torch.bfloat16, device="cuda")
    dop = {"name": "d", "kind": "Custom", "inputs": [], "outputs": [],
           "attrs": {"custom_name": "attn_decode", "params": prm}}
    of.launch(dop, [cur, kc, vc, torch.from_numpy(table).cuda(), torch.from_numpy(ctx).cuda()], [out], B)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for b, L in enumerate(lens):
        full = tb(seqs[b]).float().cpu().numpy()  # the bf16 values the GPU saw
        want = oracle.attn_prefill(full, nq, nkv, hd, L + 1)[-1]
        assert rel_err(got[b], want) < 1e-2, (b, L, rel_err(got[b], want))
