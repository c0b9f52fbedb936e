python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02j_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02j_gpu_tests.log 2>&1
timeout 600 python bench.py --entries 2048 --no-cpu-baseline --no-e2e > gpurun_out/r02j_2048.json 2> gpurun_out/r02j_2048.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02j_w5.json 2> gpurun_out/r02j_w5.err
