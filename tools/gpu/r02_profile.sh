# round-2 evidence: launch list of the prefill bench leg (4 layers) and ncu --set full of the hot kernels
set -x
NCU="ncu --clock-control none"
timeout 900 $NCU --metrics gpu__time_duration.sum -c 3000 --csv --log-file gpurun_out/r02_launches_prefill4.csv \
  python bench.py --layers 4 --no-decode --no-moe --no-toy --no-cpu --steps 2 --warmup 1 --rounds 1 --soak 0 > gpurun_out/r02_launches_prefill4.log 2>&1; echo "launches rc=$?"
timeout 900 $NCU --metrics gpu__time_duration.sum -c 3000 --csv --log-file gpurun_out/r02_launches_decode4.csv \
  python bench.py --layers 4 --workload prefill --no-moe --no-toy --no-cpu --steps 2 --warmup 1 --rounds 1 --soak 0 --sm-sweep > gpurun_out/r02_launches_decode4.log 2>&1; echo "launches2 rc=$?"
timeout 900 $NCU --set full --import-source on -o gpurun_out/r02_full_all python tools/profile_kernels.py all > gpurun_out/r02_full_all.log 2>&1; echo "full rc=$?"
timeout 600 $NCU --set full --import-source on -o gpurun_out/r02_full_tp8 python tools/profile_kernels.py proj_tp8 > gpurun_out/r02_full_tp8.log 2>&1; echo "tp8 rc=$?"
ls -la gpurun_out
