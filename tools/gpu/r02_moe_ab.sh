#!/bin/bash
# MoE grouped-GEMM epilogue A/B (HEAD gemm.cu vs working tree), then MoE parity tests
set -u
mkdir -p gpurun_out
for r in 1 2 3; do
  OPF_LIB=paper_2605_21603_b200/libopflow_b200_HEAD.so timeout 300 python tools/moe_ab.py >> gpurun_out/moe_ab.jsonl 2>>gpurun_out/moe_ab.err
  timeout 300 python tools/moe_ab.py >> gpurun_out/moe_ab.jsonl 2>>gpurun_out/moe_ab.err
done
timeout 600 python -m pytest -q -x tests/test_gpu_moe.py tests/test_gpu_moe_ep.py tests/test_gpu_fullsize.py > gpurun_out/moe_tests.log 2>&1; echo "moe tests rc=$?"; tail -2 gpurun_out/moe_tests.log
