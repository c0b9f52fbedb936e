timeout 900 python -m pytest tests/test_gpu_hull.py tests/test_gpu_parity.py tests/test_gpu_f2.py tests/test_gpu_f3.py -q -k "f64 or fp64 or frontier or gamma or f2 or a7" > gpurun_out/f64c_tests.log 2>&1
timeout 900 python tools/prof_f64.py > gpurun_out/f64c.log 2>&1
