timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "accum_full_size" > gpurun_out/acctest.log 2>&1
