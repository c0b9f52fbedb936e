timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "expected or eval" > gpurun_out/w4b_tests.log 2>&1
timeout 600 python bench.py --workload W4 --no-cpu-baseline --no-e2e > gpurun_out/w4b_bench.json 2> gpurun_out/w4b_bench.err
timeout 600 python tools/prof_eval.py --sweep > gpurun_out/w4b_prof_eval.log 2>&1
