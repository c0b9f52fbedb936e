for i in 1 2; do
  (cd ab_old && timeout 300 python tools/prof_dp.py --entries 16384 --reps 3) > gpurun_out/h_old_$i.log 2>&1
  timeout 300 python tools/prof_dp.py --entries 16384 --reps 3 > gpurun_out/h_new_$i.log 2>&1
done
