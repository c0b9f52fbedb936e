python -c "from paper_2605_05219_b200 import build as b; b.build()" > gpurun_out/big_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hull.py -q > gpurun_out/big_hulltest.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/big_gputest.log 2>&1
timeout 600 python tools/prof_dp.py --entries 16384 --reps 3 > gpurun_out/big_prof.log 2>&1
timeout 600 python tools/prof_dp.py --entries 4096 --reps 2 --plus1 >> gpurun_out/big_prof.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dp_hull_kernel -s 3 -c 1 \
  -o gpurun_out/big_ones python tools/prof_dp.py --entries 2048 --reps 2 --plus1 > gpurun_out/big_ones_ncu.log 2>&1
