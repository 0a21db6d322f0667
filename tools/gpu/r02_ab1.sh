set -x
timeout 900 python -m pytest tests/test_gpu_moe.py tests/test_gpu_moe_ep.py tests/test_gpu_multiproc.py -x -q -p no:cacheprovider > gpurun_out/r02_ab1_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_ab1_pytest.log
export AB_SHAPES=8192x768x4096,8192x4096x512,8192x3584x4096,8192x4096x1792,8192x6144x4096,8192x4096x4096,512x4096x4096,512x28672x4096
for r in 1 2; do
  OPF_LIB=paper_2605_21603_b200/libopflow_b200_HEAD.so timeout 300 python tools/gemm_ab.py >> gpurun_out/r02_ab1_gemm.jsonl 2>>gpurun_out/r02_ab1_gemm.err
  timeout 300 python tools/gemm_ab.py >> gpurun_out/r02_ab1_gemm.jsonl 2>>gpurun_out/r02_ab1_gemm.err
done
OPF_LIB=paper_2605_21603_b200/_build/libopflow_trace.so timeout 120 python tools/gemm_trace.py 8192 4096 512 > gpurun_out/r02_ab1_trace_o.txt 2>&1
timeout 600 python bench.py --layers 2 --no-decode --no-toy --no-cpu --steps 5 > gpurun_out/r02_ab1_bench.json 2>gpurun_out/r02_ab1_bench.err; echo "bench rc=$?"
