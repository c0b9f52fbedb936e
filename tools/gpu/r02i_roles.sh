for i in 1 2; do
  timeout 300 python tools/prof_dp.py --entries 2048 --reps 3 > gpurun_out/ro_main_$i.log 2>&1
  (cd ab_new && timeout 300 python tools/prof_dp.py --entries 2048 --reps 3) > gpurun_out/ro_new_$i.log 2>&1
done
(cd ab_new && timeout 900 python -m pytest tests/test_gpu_hull.py tests/test_gpu_parity.py -q -x -p no:cacheprovider) > gpurun_out/ro_new_tests.log 2>&1
