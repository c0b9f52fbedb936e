# int64 / fp64 hull kernels capped at 168 registers (9 warps/SM, smem-bound) vs default (8: the
# 202 / 192-register warps fit 2 per SM sub-partition)
for i in 1 2; do
  timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000 > gpurun_out/mb_main_acc_$i.log 2>&1
  (cd ab_new && timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000) > gpurun_out/mb_new_acc_$i.log 2>&1
done
timeout 600 python tools/prof_f64.py > gpurun_out/mb_main_f64.log 2>&1
(cd ab_new && timeout 600 python tools/prof_f64.py) > gpurun_out/mb_new_f64.log 2>&1
(cd ab_new && timeout 900 python -m pytest tests/test_gpu_hull.py tests/test_gpu_parity.py -q -x -k "int64 or f64 or fp64 or huge or accum or large" -p no:cacheprovider) > gpurun_out/mb_new_tests.log 2>&1
