set -x
export OPF_LIB=paper_2605_21603_b200/_build/libopflow_trace.so
timeout 120 python tools/gemm_trace.py 512 6144 4096 rope > gpurun_out/r02_trace_qkv512_rope.txt 2>&1
timeout 120 python tools/gemm_trace.py 512 6144 4096 > gpurun_out/r02_trace_qkv512.txt 2>&1
timeout 120 python tools/gemm_trace.py 8192 6144 4096 rope > gpurun_out/r02_trace_qkv8192_rope.txt 2>&1
unset OPF_LIB
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r02_launches_step_prefill4.csv python tools/replay_step.py prefill 4 > gpurun_out/r02_launches_step.log 2>&1; echo "ncu rc=$?"
