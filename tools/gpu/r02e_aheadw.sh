for i in 1 2; do
  timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000 > gpurun_out/aw_main_acc_$i.log 2>&1
  (cd variants/aheadw && timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000) > gpurun_out/aw_new_acc_$i.log 2>&1
done
timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --f64 > gpurun_out/aw_main_f64.log 2>&1
(cd variants/aheadw && timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --f64) > gpurun_out/aw_new_f64.log 2>&1
