"""GPU: the peer-memory collectives (one-shot all-reduce, fused all-reduce +
residual add + RMSNorm) run their full cross-rank flag protocol with W
"virtual ranks" sharing one B200 (each rank = its own window, launch and
stream).  The real multi-GPU path differs only in how the windows are mapped
(CUDA IPC over NVLink instead of same-device pointers)."""
import numpy as np
import pytest

from oracle import oracle
from paper_2605_21603_b200 import opflow as of
from paper_2605_21603_b200.workloads import rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("built")]


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("ar_mode,rows", [(0, 64), (1, 64), (2, 64), (2, 61), (3, 64), (3, 61)])
def test_fused_allreduce_add_rmsnorm_virtual_ranks(cuda, world, ar_mode, rows):
    """ar_mode 1: one-shot, pull form (every rank reads every rank's rows);
    3: one-shot, push form (every rank writes its rows into every peer's
    window; the default when the window holds world planes, else mode 1);
    2: two-shot (reduce-scatter by row blocks -> add + norm -> all-gather);
    0: automatic.  Includes a row count that does not divide by the world size."""
    import torch
    H = 4096
    comms = of.Comm.virtual(world, 0, max(3, world if ar_mode == 3 else 3) * rows * H * 2)
    rng = np.random.default_rng(world)
    tb = lambda a: torch.from_numpy(a.astype(np.float32)).cuda().to(torch.bfloat16)
    x = tb(rng.uniform(-1, 1, (rows, H)))
    g = tb(1 + 0.1 * rng.uniform(-1, 1, H))
    streams = [torch.cuda.Stream() for _ in range(world)]
    op = {"name": "f", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "allreduce_add_rmsnorm", "world_size": world,
                    "params": {"eps": 1e-5, "ar_mode": ar_mode}}}
    for it in range(3):  # epochs advance on the device across calls
        parts = [tb(rng.uniform(-1, 1, (rows, H))) for _ in range(world)]
        outs = [(torch.empty_like(x), torch.empty_like(x)) for _ in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            of.launch(op, [parts[r], x, g], list(outs[r]), rows, streams[r], comm=comms[r], max_ctas=8)
        torch.cuda.synchronize()
        for c in comms:
            assert c.window_error() == 0
        s = x.float().cpu().numpy() + sum(p.float().cpu().numpy() for p in parts)
        want_h = oracle.rmsnorm(s, g.float().cpu().numpy(), 1e-5)
        for r in range(world):
            assert rel_err(outs[r][0].float().cpu().numpy(), s) < 1e-2
            assert rel_err(outs[r][1].float().cpu().numpy(), want_h) < 1e-2
    # one-shot all-reduce (the AllReduce kind with a windowed communicator)
    ar = {"name": "ar", "kind": "AllReduce", "inputs": [], "outputs": [], "attrs": {"world_size": world}}
    parts = [tb(rng.uniform(-1, 1, (rows, H))) for _ in range(world)]
    outs = [torch.empty_like(x) for _ in range(world)]
    torch.cuda.synchronize()
    for r in range(world):
        of.launch(ar, [parts[r]], [outs[r]], rows, streams[r], comm=comms[r], max_ctas=8)
    torch.cuda.synchronize()
    want = sum(p.float().cpu().numpy() for p in parts)
    for r in range(world):
        assert rel_err(outs[r].float().cpu().numpy(), want) < 1e-2


@pytest.mark.parametrize("ar_mode", [1, 2, 3])
def test_barrier_epochs_wrap_around(cuda, ar_mode):
    """Epochs and flags are u32 that grow forever in device memory; seeded just
    below 2^32, twenty calls cross the wrap.  The barrier compares in serial-
    number order, so every call still waits for its peers (right results, no
    timeout) — an unsigned `<` would let a rank run ahead after the wrap."""
    import torch
    world, rows, H = 2, 64, 4096
    comms = of.Comm.virtual(world, 0, 3 * rows * H * 2)
    for c in comms:
        c.set_epochs(0xFFFFFFFF - 6)
    rng = np.random.default_rng(5)
    tb = lambda a: torch.from_numpy(a.astype(np.float32)).cuda().to(torch.bfloat16)
    x = tb(rng.uniform(-1, 1, (rows, H)))
    g = tb(1 + 0.1 * rng.uniform(-1, 1, H))
    streams = [torch.cuda.Stream() for _ in range(world)]
    op = {"name": "f", "kind": "Custom", "inputs": [], "outputs": [],
          "attrs": {"custom_name": "allreduce_add_rmsnorm", "world_size": world,
                    "params": {"eps": 1e-5, "ar_mode": ar_mode}}}
    for it in range(20):
        parts = [tb(rng.uniform(-1, 1, (rows, H))) for _ in range(world)]
        outs = [(torch.empty_like(x), torch.empty_like(x)) for _ in range(world)]
        torch.cuda.synchronize()
        for r in range(world):
            of.launch(op, [parts[r], x, g], list(outs[r]), rows, streams[r], comm=comms[r], max_ctas=8)
        torch.cuda.synchronize()
        s = x.float().cpu().numpy() + sum(p.float().cpu().numpy() for p in parts)
        for r in range(world):
            assert rel_err(outs[r][0].float().cpu().numpy(), s) < 1e-2, (it, r)
    for c in comms:
        assert c.window_error() == 0
