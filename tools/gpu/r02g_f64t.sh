timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "f64" > gpurun_out/f64t.log 2>&1
