#!/bin/bash
# round-2 final evidence: GPU suite, smoke, bench (ours + reference arm), launch lists, ncu --set full captures
set -x
mkdir -p gpurun_out/final gpurun_out/final/ncu
O=gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum -c 3000 --csv --log-file $O/launches_prefill4.csv \
  python bench.py --layers 4 --no-decode --no-moe --no-toy --no-cpu --steps 2 --warmup 1 --rounds 1 --soak 0 > $O/launches_prefill4.log 2>&1; echo "launches rc=$?"
timeout 600 $NCU --metrics gpu__time_duration.sum -c 600 --csv --log-file $O/launches_decode4.csv \
  python tools/step_breakdown.py decode 4 > $O/launches_decode4.log 2>&1; echo "launches2 rc=$?"
cap() {  # name, which, kernel regex, count
  timeout 400 $NCU --set full --import-source on -f -k "regex:$3" -c $4 -o /tmp/$1 python tools/profile_kernels.py $2 > $O/ncu/$1.log 2>&1
  echo "$1 rc=$?"
  python profiles/ncu_summary.py /tmp/$1.ncu-rep > $O/ncu/$1.summary.txt 2>&1
  ncu -i /tmp/$1.ncu-rep --page details --csv > $O/ncu/$1.details.csv 2>/dev/null
}
cap r02f_proj proj gemm_tc2 4
cap r02f_tp8 proj_tp8 gemm_tc2 4
cap r02f_prefill prefill fa_ 1
cap r02f_decode decode decode_t 1
cap r02f_norm norm rmsnorm 1
cap r02f_moe moe "gemm_tc|gather|combine|route|topk" 10
du -sh gpurun_out
