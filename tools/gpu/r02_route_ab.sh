#!/bin/bash
# MoE routing-kernel A/B (HEAD moe.cu vs working tree) + MoE / EP parity
timeout 400 python -m pytest -q -x tests/test_gpu_moe.py tests/test_gpu_moe_ep.py tests/test_gpu_multiproc.py 2>&1 | tail -2
for i in 1 2 3; do
  OPF_LIB=paper_2605_21603_b200/libopflow_b200_HEAD.so timeout 200 python tools/moe_ab.py | sed 's/^/HEAD /'
  timeout 200 python tools/moe_ab.py | sed 's/^/NEW  /'
done
