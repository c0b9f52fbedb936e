timeout 900 python -m pytest tests/test_gpu_hull.py -q > gpurun_out/big3_hulltest.log 2>&1
for i in 1 2; do
  (cd ab_old && timeout 300 python tools/prof_dp.py --entries 16384 --reps 3) > gpurun_out/ab3_old_$i.log 2>&1
  timeout 300 python tools/prof_dp.py --entries 16384 --reps 3 > gpurun_out/ab3_new_$i.log 2>&1
done
timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --ones > gpurun_out/ab3_ones.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dp_hull_kernel -s 2 -c 1 \
  -o gpurun_out/big_ones python tools/prof_dp.py --entries 2048 --reps 2 --ones > gpurun_out/big_ones_ncu.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/big3_gputest.log 2>&1
