set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_ref.json 2>gpurun_out/r02_bench_ref.err; echo "ref rc=$?"
tail -c 1500 gpurun_out/r02_bench_ref.json
