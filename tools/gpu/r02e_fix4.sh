timeout 900 python -m pytest tests/test_gpu_hull.py -q > gpurun_out/fix4_tests.log 2>&1
