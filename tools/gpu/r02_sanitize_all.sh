#!/bin/bash
# memcheck over the whole GPU suite except the virtual-rank EP tests (their cross-"rank" barriers
# need concurrent kernels, which the tool serialises: they fail on window_error by design) and the
# multi-process tests (run under the tool through OPF_MP_WRAP, separately)
mkdir -p gpurun_out/san
timeout 3000 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -m gpu tests \
  --deselect tests/test_gpu_moe_ep.py --ignore=tests/test_gpu_moe_ep.py --ignore=tests/test_gpu_multiproc.py \
  > gpurun_out/san/memcheck_all.log 2>&1; echo "memcheck rc=$?"
grep -E "passed|failed|ERROR SUMMARY" gpurun_out/san/memcheck_all.log | tail -5
OPF_MP_WRAP="compute-sanitizer --tool memcheck" timeout 1500 python -m pytest -q -x tests/test_gpu_multiproc.py \
  > gpurun_out/san/memcheck_multiproc.log 2>&1; echo "mp rc=$?"; tail -2 gpurun_out/san/memcheck_multiproc.log
