for i in 1 2; do
  timeout 300 python tools/prof_dp.py --entries 16384 --reps 3 > gpurun_out/op_main_$i.log 2>&1
  (cd ab_new && timeout 300 python tools/prof_dp.py --entries 16384 --reps 3) > gpurun_out/op_new_$i.log 2>&1
done
(cd ab_new && timeout 900 python -m pytest tests/test_gpu_hull.py tests/test_gpu_parity.py -q -x -k "w5 or hull or small or edge" -p no:cacheprovider) > gpurun_out/op_new_tests.log 2>&1
