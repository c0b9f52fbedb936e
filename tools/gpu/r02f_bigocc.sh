timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --ones > gpurun_out/bo_main.log 2>&1
for v in 2048 4096; do (cd ab_p$v && timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --ones) > gpurun_out/bo_$v.log 2>&1; done
