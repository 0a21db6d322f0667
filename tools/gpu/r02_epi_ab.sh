#!/bin/bash
# GEMM epilogue A/B: swizzled smem staging + coalesced 16B stores (default) vs per-lane 256-bit stores (OPF_EPI_DIRECT)
export AB_SHAPES=8192x4096x512,8192x768x4096,8192x3584x4096,8192x4096x1792,8192x4096x4096,8192x28672x4096,8192x4096x14336,512x4096x4096
for i in 1 2; do
  timeout 200 python tools/gemm_ab.py
  OPF_LIB=paper_2605_21603_b200/_build/libopflow_epidirect.so timeout 200 python tools/gemm_ab.py
done
for i in 1 2; do
  echo "BASE $(timeout 200 python tools/prefill_ab.py 8 2>/dev/null | tail -1)"
  echo "DIRECT $(OPF_LIB=paper_2605_21603_b200/_build/libopflow_epidirect.so timeout 200 python tools/prefill_ab.py 8 2>/dev/null | tail -1)"
done
