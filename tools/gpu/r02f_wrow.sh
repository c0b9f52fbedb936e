for i in 1 2; do
  timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000 > gpurun_out/wr_main_acc_$i.log 2>&1
  (cd ab_new && timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000) > gpurun_out/wr_new_acc_$i.log 2>&1
done
timeout 600 python tools/prof_f64.py > gpurun_out/wr_main_f64.log 2>&1
(cd ab_new && timeout 600 python tools/prof_f64.py) > gpurun_out/wr_new_f64.log 2>&1
