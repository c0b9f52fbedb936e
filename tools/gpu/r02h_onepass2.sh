for i in 1 2; do
  timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000 > gpurun_out/o2_main_acc_$i.log 2>&1
  (cd ab_new && timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --dense-n 120000 180000) > gpurun_out/o2_new_acc_$i.log 2>&1
done
timeout 600 python tools/prof_f64.py > gpurun_out/o2_main_f64.log 2>&1
(cd ab_new && timeout 600 python tools/prof_f64.py) > gpurun_out/o2_new_f64.log 2>&1
for w in W3 W2; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 20 >> gpurun_out/o2_main_small.jsonl 2>/dev/null
  (cd ab_new && cp ../bench.py . && timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 20) >> gpurun_out/o2_new_small.jsonl 2>/dev/null
done
(cd ab_new && timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider) > gpurun_out/o2_new_tests.log 2>&1
