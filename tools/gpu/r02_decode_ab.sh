set -x
timeout 1200 python tools/decode_ab.py --layers 8 --reps 2 --sms 40,56 --var ef: --var normal:OPF_DECODE_L2=normal > gpurun_out/r02_decode_ab.log 2>&1; echo "ab rc=$?"
tail -5 gpurun_out/r02_decode_ab.log
