# W4 budget sweep CSV; fp64 DP timing on W5 rows (w = c / n)
timeout 600 python tools/budget_sweep.py --out gpurun_out/r02e_w4_sweep.csv > gpurun_out/r02e_w4_sweep.log 2>&1
timeout 900 python tools/prof_dp.py --entries 16384 --reps 3 --f64 > gpurun_out/r02e_f64.log 2>&1
timeout 900 python tools/prof_dp.py --entries 16384 --reps 3 >> gpurun_out/r02e_f64.log 2>&1
