for i in 1 2; do
  timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --ones > gpurun_out/bop_main_$i.log 2>&1
  (cd ab_new && timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --ones) > gpurun_out/bop_new_$i.log 2>&1
done
(cd ab_new && timeout 900 python -m pytest tests/test_gpu_hull.py -q -x -p no:cacheprovider) > gpurun_out/bop_new_tests.log 2>&1
