# large-hull mode: its tests, the whole GPU suite, the all-ones and W5 bench lines
python -c "from paper_2605_05219_b200 import build as b; b.build()" > gpurun_out/big_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hull.py -x -q > gpurun_out/big_hulltest.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/big_gputest.log 2>&1
timeout 600 python bench.py --dp-hist ones --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/big_ones.json 2> gpurun_out/big_ones.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/big_w5.json 2> gpurun_out/big_w5.err
