#!/bin/bash
# fast-reciprocal SiLU epilogue A/B (HEAD gemm.cu vs working tree): prefill + decode legs, 8 layers
timeout 300 python -m pytest -q -x tests/test_gpu_fusion.py tests/test_gpu_moe.py 2>&1 | tail -1
for i in 1 2 3; do
  echo "HEAD $(OPF_LIB=paper_2605_21603_b200/libopflow_b200_HEAD.so timeout 200 python tools/prefill_ab.py 8 2>/dev/null | tail -1)"
  echo "NEW  $(timeout 200 python tools/prefill_ab.py 8 2>/dev/null | tail -1)"
done
timeout 600 python tools/decode_ab.py --layers 8 --reps 2 --sms "" --var head:OPF_LIB=paper_2605_21603_b200/libopflow_b200_HEAD.so --var new: 2>&1 | tail -1
