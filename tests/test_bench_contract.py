"""CPU: bench.py's driver contract — the reference arm's JSON line (same metric
and config keys as ours, CPU baseline fields, no GPU transfers) and the
refusal to run a smaller tensor-parallel degree than --gpus asks for."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(*args, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=env, capture_output=True,
                          text=True, timeout=timeout)


def test_gpus_n_without_gpus_fails_loudly():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("GPUs present: --gpus 2 would really launch two ranks")
    r = _run("--gpus", "2", "--steps", "1", "--warmup", "0", timeout=300)
    assert r.returncode == 2, (r.returncode, r.stderr[-500:])
    assert "refusing" in r.stderr


def test_reference_arm_line():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    r = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert r.returncode == 0, r.stderr[-800:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    import bench
    assert line["metric"] == bench.METRIC and line["unit"] == "tokens/s" and line["higher_is_better"] is True
    # one replica of 8192 tokens whatever N is (TP=N shards the layer): total work fixed
    assert line["scaling"] == "strong"
    assert line["config"]["workload"].startswith("llama3-8b-shaped prefill, 32 layers, 8192 tokens")
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] > 0 and cb["cpu_model"]
    assert line["e2e"] == {"value": line["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
