timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hull.py tests/test_gpu_f2.py tests/test_gpu_f3.py -q -x -k "f64 or fp64 or frontier or gamma or f2 or a7 or expected" > gpurun_out/f64d_tests.log 2>&1
timeout 900 python tools/prof_f64.py > gpurun_out/f64d.log 2>&1
timeout 900 python bench.py --weights f64 --no-cpu-baseline > gpurun_out/f64d_bench.json 2> gpurun_out/f64d_bench.err
