for i in 1 2; do
  timeout 300 python tools/prof_dp.py --entries 16384 --reps 3 > gpurun_out/lp_main_$i.log 2>&1
  (cd ab_new && timeout 300 python tools/prof_dp.py --entries 16384 --reps 3) > gpurun_out/lp_new_$i.log 2>&1
done
timeout 300 python tools/prof_dp.py --entries 2048 --reps 3 > gpurun_out/lp_main_2048.log 2>&1
(cd ab_new && timeout 300 python tools/prof_dp.py --entries 2048 --reps 3) > gpurun_out/lp_new_2048.log 2>&1
timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000 > gpurun_out/lp_main_acc.log 2>&1
(cd ab_new && timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000) > gpurun_out/lp_new_acc.log 2>&1
