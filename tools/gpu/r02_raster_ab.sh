#!/bin/bash
# GEMM raster A/B (group_m x reversed-K on odd tiles): timing + ncu DRAM bytes
set -u
mkdir -p gpurun_out
export AB_SHAPES=8192x6144x4096,8192x4096x4096,8192x28672x4096,8192x4096x14336,8192x3584x4096,8192x4096x1792
for round in 1 2; do
  for v in "16 0" "16 1" "32 0" "32 1" "8 1"; do
    set -- $v
    OPF_GEMM_GROUP=$1 OPF_GEMM_REVK=$2 timeout 300 python tools/gemm_ab.py >> gpurun_out/raster_ab.jsonl 2>> gpurun_out/raster_ab.err
  done
done
for v in "16 0" "16 1" "32 0" "32 1"; do
  set -- $v
  OPF_GEMM_GROUP=$1 OPF_GEMM_REVK=$2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:gemm_tc2 --csv python tools/profile_kernels.py proj > gpurun_out/raster_ncu_g$1_r$2.csv 2>/dev/null
done
