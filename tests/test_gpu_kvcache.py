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


def test_two_step_decode_loop_through_the_engine(cuda):
    """A serving loop: two decode steps of llama_decode_graph(kv_write=1) over
    manager-owned HND page pools.  Step 1 appends each sequence's token to the
    cache; step 2 attends over it.  Both steps' outputs match the oracle, which
    carries its own caches across the steps (its kv_write semantics)."""
    import torch
    from paper_2605_21603_b200.workloads import llama_inputs
    B, ctx_max, page, layers = 6, 64, 16, 2
    shape = dict(layers=layers, tokens=B, hidden=256, heads=4, kv_heads=2, head_dim=128, inter=512,
                 ctx_len=ctx_max, page_size=page, dtype="bf16", kv_layout=1, kv_write=1, num_pages=40)
    desc = of.llama_decode_graph(**shape)
    kv = of.KvCache(layers=layers, pages=40, kv_heads=2, head_dim=128, page_size=page, kv_layout=1)
    lens = [3, 15, 16, 17, 30, 47]
    kv.append(list(range(B)), lens)  # prompt pages, filled with random K / V below
    host = llama_inputs(desc, B, seed=31, ctx_len=8)
    g = of.build_graph(desc)
    sess = of.Session(g, of.partition(g, [of.PartitionRule.by_func("attn_decode")]), {"lanes": 3})
    keep = {}
    rng = np.random.default_rng(3)
    for l in range(layers):
        for w in ("k", "v"):
            t = kv.cache(l, w)
            t.copy_(torch.from_numpy(rng.uniform(-1, 1, t.shape).astype(np.float32)).to(torch.bfloat16))
            keep[f"layer{l}.{w}_cache"] = t
    for t in g.description["tensors"]:
        n = t["name"]
        if t["role"] == "weight" and n not in keep:
            keep[n] = torch.from_numpy(host[n]).cuda().to(torch.bfloat16)
    for n, t in keep.items():
        sess.bind(n, t)
    out = torch.empty(B, shape["hidden"], dtype=torch.bfloat16, device="cuda")
    out_name = [t["name"] for t in g.description["tensors"] if t["role"] == "output" and t.get("dtype") != "i64"][0]
    sess.bind(out_name, out)
    oracle_caches = {n: v.float().cpu().numpy() for n, v in keep.items() if n.endswith("_cache")}
    for step in range(2):
        slots, pos = kv.append(list(range(B)), [1] * B)
        table, _ = kv.block_table(list(range(B)), ctx_max // page)
        table = np.where(table < 0, 0, table)
        x = rng.uniform(-1, 1, (B, shape["hidden"])).astype(np.float32)
        step_in = {"x": torch.from_numpy(x).cuda().to(torch.bfloat16), "positions": torch.from_numpy(pos).cuda(),
                   "slots": torch.from_numpy(slots).cuda(), "block_table": torch.from_numpy(table).cuda()}
        for n, v in step_in.items():
            keep[n] = v
            sess.bind(n, v)
        sess.run({"name": "split_overlap", "n_microbatches": 2, "lane_mode": "ubatch"})
        torch.cuda.synchronize()
        ohost = dict(host)
        ohost.update({n: v for n, v in oracle_caches.items()})
        ohost.update({"x": step_in["x"].float().cpu().numpy(), "positions": pos, "slots": slots, "block_table": table})
        for n in ohost:
            if n.endswith(".w"):
                ohost[n] = keep[n].float().cpu().numpy()
        new_caches = {}
        want = oracle.evaluate(desc, B, ohost, exact=False, caches_out=new_caches)
        oracle_caches.update(new_caches)
        err = rel_err(out.float().cpu().numpy(), want[out_name])
        assert err < 2e-2, (step, err)


def test_prefill_then_decode_equals_longer_prefill(cuda):
    """End to end over every layer: a prefill graph (kv_write=1) fills the
    paged caches for B prompts of S tokens, then one decode step (kv_write=1)
    on token S; its output must equal the last row of a plain prefill over the
    S + 1 tokens (causal attention), layer stack and all."""
    import torch
    from paper_2605_21603_b200.workloads import llama_inputs
    B, S, layers, page, pages = 3, 16, 2, 16, 24
    base = dict(layers=layers, hidden=256, heads=4, kv_heads=2, head_dim=128, inter=512, dtype="bf16")
    pre = of.llama_graph(tokens=B * S, seq_len=S, kv_write=1, num_pages=pages, kv_layout=1, page_size=page, **base)
    dec = of.llama_decode_graph(tokens=B, ctx_len=S + page, page_size=page, kv_layout=1, kv_write=1,
                                num_pages=pages, **base)
    full = of.llama_graph(tokens=B * (S + 1), seq_len=S + 1, **base)
    w = llama_inputs(full, B * (S + 1), seed=41)
    rng = np.random.default_rng(41)
    xs = rng.uniform(-1, 1, (B, S + 1, base["hidden"])).astype(np.float32)
    tb = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.bfloat16)
    kv = of.KvCache(layers=layers, pages=pages, kv_heads=2, head_dim=128, page_size=page, kv_layout=1)
    keep = []

    def session(desc, binds):
        g = of.build_graph(desc)
        sess = of.Session(g, of.partition(g, []), {"lanes": 3})
        out = None
        for t in g.description["tensors"]:
            n = t["name"]
            if t["role"] == "output":
                if t.get("dtype") == "i64":
                    continue
                out = torch.empty(list(t["shape"]), dtype=torch.bfloat16, device="cuda")
                sess.bind(n, out)
            elif n in binds:
                sess.bind(n, binds[n])
            elif n.endswith("_cache"):
                l = int(n.split(".")[0][5:])
                sess.bind(n, kv.cache(l, "k" if n.endswith("k_cache") else "v"))
            elif t["role"] == "weight":
                v = tb(w[n])
                keep.append(v)
                sess.bind(n, v)
        keep.append(binds)
        return sess, out

    # prefill of the prompts: fills every layer's pages
    slots, pos = kv.append(list(range(B)), [S] * B)
    sp, _ = session(pre, {"x": tb(xs[:, :S].reshape(B * S, -1)), "positions": torch.from_numpy(pos).cuda(),
                          "slots": torch.from_numpy(slots).cuda()})
    sp.run({"name": "sequential"})
    # one decode step on token S
    slots, pos = kv.append(list(range(B)), [1] * B)
    table, _ = kv.block_table(list(range(B)), (S + page) // page)
    sd, out = session(dec, {"x": tb(xs[:, S]), "positions": torch.from_numpy(pos).cuda(),
                            "slots": torch.from_numpy(slots).cuda(),
                            "block_table": torch.from_numpy(np.where(table < 0, 0, table)).cuda()})
    sd.run({"name": "split_overlap", "n_microbatches": 2, "lane_mode": "ubatch"})
    # the same tokens as one causal prefill of S + 1 per sequence
    sf, ref = session(full, {"x": tb(xs.reshape(B * (S + 1), -1)),
                             "positions": torch.from_numpy((np.arange(B * (S + 1)) % (S + 1)).astype(np.int64)).cuda()})
    sf.run({"name": "sequential"})
    torch.cuda.synchronize()
    want = ref.float().view(B, S + 1, -1)[:, S].cpu().numpy()
    err = rel_err(out.float().cpu().numpy(), want)
    assert err < 2e-2, err
