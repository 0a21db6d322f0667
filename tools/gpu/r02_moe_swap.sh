#!/bin/bash
# swapped-operand grouped expert GEMM: parity first (bounded), then A/B vs the token-major kernel
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest -q -x tests/test_gpu_moe.py > gpurun_out/swap_tests.log 2>&1; rc=$?; echo "moe tests rc=$rc"; tail -15 gpurun_out/swap_tests.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 300 python -m pytest -q -x tests/test_gpu_moe_ep.py tests/test_gpu_fullsize.py > gpurun_out/swap_tests2.log 2>&1; echo "ep/fullsize rc=$?"; tail -3 gpurun_out/swap_tests2.log
for r in 1 2; do
  OPF_MOE_SWAP=0 timeout 200 python tools/moe_ab.py >> gpurun_out/swap_ab.jsonl 2>>gpurun_out/swap_ab.err
  timeout 200 python tools/moe_ab.py >> gpurun_out/swap_ab.jsonl 2>>gpurun_out/swap_ab.err
done
python - <<'P'
import json
for l in open('gpurun_out/swap_ab.jsonl'):
    d=json.loads(l); print(d['strategies_ms'], [(p['op'],p['ms']) for p in d['per_op']])
P
