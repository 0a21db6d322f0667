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
