#!/bin/bash
# ncu --set full with source of the prefill attention and the MoE grouped GEMMs (stall analysis)
NCU="ncu --clock-control none"
mkdir -p gpurun_out
timeout 600 $NCU --set full --import-source on -k regex:fa_pp -c 1 -o gpurun_out/r02s_fa python tools/profile_kernels.py prefill > gpurun_out/r02s_fa.log 2>&1; echo "fa rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:gemm_tc_kernel -c 2 -o gpurun_out/r02s_moe python tools/profile_kernels.py moe > gpurun_out/r02s_moe.log 2>&1; echo "moe rc=$?"
ls -la gpurun_out/*.ncu-rep
