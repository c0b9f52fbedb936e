timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fix2_gputest.log 2>&1
timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000 > gpurun_out/fix2_acc.log 2>&1
timeout 600 python tools/prof_f64.py >> gpurun_out/fix2_acc.log 2>&1
