for i in 1 2; do
  (cd ab_old && timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000) > gpurun_out/ab64_old_$i.log 2>&1
  timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000 > gpurun_out/ab64_new_$i.log 2>&1
done
