timeout 900 python -m pytest tests/test_gpu_hull.py -q > gpurun_out/big4_hulltest.log 2>&1
timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --ones > gpurun_out/big4_ones.log 2>&1
(cd variants/big12 && timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --ones) > gpurun_out/big4_ones12.log 2>&1
(cd variants/big12 && SP_HULL_BIG_TEST=1 timeout 900 python -m pytest ../../tests/test_gpu_hull.py -q -k "large_hull or overflow" -p no:cacheprovider) > gpurun_out/big4_hulltest12.log 2>&1
timeout 300 python tools/prof_dp.py --entries 16384 --reps 2 >> gpurun_out/big4_ones.log 2>&1
