# ncu --set full of each hot kernel (bounded: -k filter, -c count), summarised on the box;
# only reports < 12 MB are copied back (gpurun_out merge limit 64 MiB)
set -x
mkdir -p gpurun_out/ncu
NCU="ncu --clock-control none --set full --import-source on"
cap() {  # name, which, kernel regex, count
  timeout 400 $NCU -k "regex:$3" -c $4 -o /tmp/$1 python tools/profile_kernels.py $2 > gpurun_out/ncu/$1.log 2>&1
  echo "$1 rc=$?"
  python profiles/ncu_summary.py /tmp/$1.ncu-rep > gpurun_out/ncu/$1.summary.txt 2>&1
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/ncu/$1.details.csv 2>/dev/null
  sz=$(stat -c %s /tmp/$1.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -lt 12000000 ]; then cp /tmp/$1.ncu-rep gpurun_out/ncu/; fi
}
cap r02_full_proj proj gemm_tc2 4
cap r02_full_tp8 proj_tp8 gemm_tc2 4
cap r02_full_prefill prefill fa_pp 1
cap r02_full_decode decode decode_t 1
cap r02_full_norm norm rmsnorm 1
cap r02_full_moe moe "gemm_tc|gather|combine|route|topk" 10
du -sh gpurun_out
bash tools/gpu/r02_decode_ab.sh
