"""TorchDynamo frontend on the B200: a plain PyTorch Llama model compiled with
the DynaFlow backend runs through the engine (tcgen05 GEMMs, fused epilogues,
tcgen05 prefill attention) and matches the eager fp32 model within the bf16
tolerance (rel <= 2e-2), under the sequential, NanoFlow and annotated schedules."""
import pytest
import torch

from paper_2605_21603_b200 import dynamo as dyn
from torch_llama import Attention, Llama, init_

pytestmark = pytest.mark.gpu
T, S = 512, 128


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


@pytest.mark.parametrize("strategy,rules", [
    ({"name": "sequential"}, []),
    ({"name": "split_overlap", "n_microbatches": 2, "align": S, "lane_mode": "ubatch"}, []),
    ({"name": "split_overlap", "n_microbatches": 2, "align": S},
     [dyn.SplitModule(Attention), dyn.SplitFunc("silu_mul")]),
])
def test_compiled_llama_matches_eager(strategy, rules):
    ref = init_(Llama(layers=2), seed=11)
    model = init_(Llama(layers=2), seed=11).to("cuda", torch.bfloat16)
    with torch.no_grad():  # the eager fp32 reference sees the same (bf16-rounded) weights
        for p_ref, p in zip(ref.parameters(), model.parameters()):
            p_ref.copy_(p.float().cpu())
    be = dyn.backend(rules=rules, strategy=strategy)
    torch._dynamo.reset()
    fn = torch.compile(model, backend=be, fullgraph=True, dynamic=False)
    pos = (torch.arange(T) % S).to(torch.int64)
    for seed in (1, 2):  # two calls, different inputs: static buffers refreshed, graph replayed
        x = torch.rand(T, 512, generator=torch.Generator().manual_seed(seed)) * 2 - 1
        with torch.no_grad():
            got = fn(x.to("cuda", torch.bfloat16), pos.cuda())
            want = ref(x.to(torch.bfloat16).float(), pos)
        torch.cuda.synchronize()
        assert _rel(got.cpu(), want) < 2e-2
    (cg,) = be.compiled
    st = cg.sess.stats()["last"]
    assert st["captured"] and st["copied_elements"] == 0
