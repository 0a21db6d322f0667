#!/bin/bash
# compute-sanitizer on the final kernels: memcheck over the attention, GEMM / engine parity, fusion,
# kv-cache and MoE suites; racecheck + synccheck over the attention suite
mkdir -p gpurun_out/san
CS="compute-sanitizer --print-limit 20"
timeout 1500 $CS --tool memcheck python -m pytest -q -x tests/test_gpu_attention.py tests/test_gpu_parity.py \
  tests/test_gpu_fusion.py tests/test_gpu_kvcache.py tests/test_gpu_moe.py > gpurun_out/san/memcheck.log 2>&1; echo "memcheck rc=$?"
tail -5 gpurun_out/san/memcheck.log
timeout 900 $CS --tool synccheck python -m pytest -q -x tests/test_gpu_attention.py > gpurun_out/san/synccheck.log 2>&1; echo "synccheck rc=$?"
tail -3 gpurun_out/san/synccheck.log
timeout 1200 $CS --tool racecheck python -m pytest -q -x tests/test_gpu_attention.py -k "prefill" > gpurun_out/san/racecheck.log 2>&1; echo "racecheck rc=$?"
tail -3 gpurun_out/san/racecheck.log
