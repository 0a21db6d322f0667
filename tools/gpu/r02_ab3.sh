set -x
timeout 900 python -m pytest tests/test_gpu_fusion.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_kvcache.py -x -q -p no:cacheprovider > gpurun_out/r02_ab3_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_ab3_pytest.log
export AB_SHAPES=512x6144x4096xrope,8192x6144x4096xrope,8192x768x4096xrope,256x6144x4096xrope
for r in 1 2; do
  OPF_LIB=paper_2605_21603_b200/libopflow_b200_HEAD.so timeout 300 python tools/gemm_ab.py >> gpurun_out/r02_ab3_gemm.jsonl 2>>gpurun_out/r02_ab3_gemm.err
  timeout 300 python tools/gemm_ab.py >> gpurun_out/r02_ab3_gemm.jsonl 2>>gpurun_out/r02_ab3_gemm.err
done
OPF_LIB=paper_2605_21603_b200/_build/libopflow_trace.so timeout 120 python tools/gemm_trace.py 512 6144 4096 rope > gpurun_out/r02_ab3_trace_qkv512_rope.txt 2>&1
timeout 300 python tools/step_breakdown.py decode 4 > gpurun_out/r02_ab3_step_decode4.txt 2>&1
