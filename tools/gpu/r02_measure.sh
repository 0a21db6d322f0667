set -x
timeout 900 python bench.py > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err; echo "bench rc=$?"
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -c 3000 --csv --log-file gpurun_out/r02_launches_prefill4.csv \
  python bench.py --layers 4 --no-decode --no-moe --no-toy --no-cpu --steps 2 --warmup 1 --rounds 1 --soak 0 > gpurun_out/r02_launches_prefill4.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -c 600 --csv --log-file gpurun_out/r02_launches_decode4.csv \
  python tools/step_breakdown.py decode 4 > gpurun_out/r02_launches_decode4.log 2>&1; echo "launches2 rc=$?"
timeout 300 python tools/step_breakdown.py decode 4 > gpurun_out/r02_step_decode4.txt 2>&1; echo "sb rc=$?"
timeout 300 python tools/step_breakdown.py prefill 4 > gpurun_out/r02_step_prefill4.txt 2>&1; echo "sb2 rc=$?"
for shp in "8192 4096 512" "8192 768 4096" "512 4096 4096" "512 28672 4096"; do
  OPF_LIB=paper_2605_21603_b200/_build/libopflow_trace.so timeout 120 python tools/gemm_trace.py $shp > "gpurun_out/r02_gemm_trace_${shp// /x}.txt" 2>&1
done
du -sh gpurun_out
