"""Host-side GEMM planning (no GPU): the split-K decision of the tcgen05 GEMM
and the engine workspace it requests (148-SM B200 model)."""
import json

from paper_2605_21603_b200 import _lib
from paper_2605_21603_b200 import opflow as of


def splits(m, n, k, sms=0):
    return _lib.lib().opf_gemm_splits(m, n, k, sms)


def test_splitk_only_for_underfilled_grids():
    # prefill projections at TP=1 fill 74 clusters many times over: no split
    for (n, k) in [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]:
        assert splits(8192, n, k) == 1
    # decode (M = 512 / 256 nano-batch): split only when all units fit one
    # round of the 74 clusters
    assert splits(512, 4096, 4096) == 2
    assert splits(512, 4096, 14336) == 2
    assert splits(256, 4096, 14336) == 4
    assert splits(256, 6144, 4096) == 3
    # multi-round grids stay unsplit (measured slower: fixup paid by every unit)
    assert splits(512, 6144, 4096) == 1
    assert splits(8192, 768, 4096) == 1
    assert splits(256, 28672, 4096) == 1
    # 1-SM path (M <= 128) and short K never split
    assert splits(128, 4096, 4096) == 1
    assert splits(512, 4096, 256) == 1


def test_splitk_respects_sm_budget():
    # the model counts rounds over the budgeted clusters: 148 SMs -> 74 clusters
    # hold 64 units of the decode O projection in one round (S = 2); a 16-SM
    # budget (8 clusters) already has 4 rounds of whole tiles and stays unsplit
    assert splits(512, 4096, 4096, 148) == 2
    assert splits(512, 4096, 4096, 64) == 1  # 32 tiles > 32 clusters / 2
    for b in (8, 24, 40, 72, 148):
        assert 1 <= splits(512, 4096, 4096, b) <= 8


def test_splitk_workspace_planned_in_arena():
    desc = json.dumps({"tensors": [{"name": "a", "shape": [256, 4096], "dtype": "bf16", "role": "input"},
                                   {"name": "w", "shape": [4096, 6144], "batch": "replicated", "dtype": "bf16",
                                    "role": "weight"},
                                   {"name": "c", "shape": [256, 6144], "dtype": "bf16", "role": "output"}],
                       "operators": [{"name": "mm", "kind": "MatMul", "inputs": ["a", "w"], "outputs": ["c"]}]})
    g = of.build_graph(desc)
    plan = of.partition(g, [])
    _, stats = of.dry_run(g, plan, "sequential", rows=256)
    tiles, S = 24, 3
    need = tiles * S * 16 * 32 * 128 * 4 + tiles * 16 * 4
    assert stats["last"]["plan_arena_bytes"] >= need
