#!/bin/bash
# GEMM epilogue stores with L1::no_allocate (variant) vs default; attention with no_allocate (working tree)
timeout 300 python -m pytest -q -x tests/test_gpu_attention.py 2>&1 | tail -1
export AB_SHAPES=8192x6144x4096xrope,8192x4096x4096,8192x28672x4096,8192x4096x14336,8192x768x4096,8192x4096x512,8192x3584x4096,8192x4096x1792,512x28672x4096
for i in 1 2; do
  timeout 200 python tools/gemm_ab.py
  OPF_LIB=paper_2605_21603_b200/_build/libopflow_gemmna.so timeout 200 python tools/gemm_ab.py
done
for i in 1 2; do
  echo "BASE $(timeout 200 python tools/prefill_ab.py 8 2>/dev/null | tail -1)"
  echo "NA   $(OPF_LIB=paper_2605_21603_b200/_build/libopflow_gemmna.so timeout 200 python tools/prefill_ab.py 8 2>/dev/null | tail -1)"
done
for i in 1 2; do timeout 100 python tools/attn_time.py 2>/dev/null | head -1; done
