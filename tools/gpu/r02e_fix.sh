timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/fix_gputest.log 2>&1
timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000 > gpurun_out/fix_acc.log 2>&1
timeout 300 python tools/prof_dp.py --entries 16384 --reps 3 >> gpurun_out/fix_acc.log 2>&1
