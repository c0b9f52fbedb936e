python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02g_final_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02g_final_gpu_tests.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02g_final_bench.json 2> gpurun_out/r02g_final_bench.err
