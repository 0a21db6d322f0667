#!/bin/bash
# prefill attention A/B (HEAD attention_fa_tc.cu vs working tree) + parity + timeline
timeout 300 python -m pytest -q -x tests/test_gpu_attention.py 2>&1 | tail -2
for i in 1 2 3; do
  OPF_LIB=paper_2605_21603_b200/libopflow_b200_HEAD.so timeout 100 python tools/attn_time.py | head -1 | sed 's/^/HEAD /'
  timeout 100 python tools/attn_time.py | head -1 | sed 's/^/NEW  /'
done
for s in 2048 4096; do
  S=$s SEQS=$((8192/s)) OPF_LIB=paper_2605_21603_b200/libopflow_b200_HEAD.so timeout 100 python tools/attn_time.py | head -1 | sed "s/^/HEAD S=$s /"
  S=$s SEQS=$((8192/s)) timeout 100 python tools/attn_time.py | head -1 | sed "s/^/NEW  S=$s /"
done
timeout 60 ./tools/fa_pp_trace.bin > gpurun_out/fa_pp_trace.txt 2>&1
