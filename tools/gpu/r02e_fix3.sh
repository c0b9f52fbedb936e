timeout 900 python -m pytest tests/test_gpu_hull.py tests/test_gpu_parity.py -q -k "handoff or expected or eval" > gpurun_out/fix3_tests.log 2>&1
for w in W4 W3; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e >> gpurun_out/fix3_bench.jsonl 2>> gpurun_out/fix3_bench.err; done
timeout 600 python bench.py --no-cpu-baseline --no-e2e >> gpurun_out/fix3_bench.jsonl 2>> gpurun_out/fix3_bench.err
