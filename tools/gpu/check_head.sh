set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c1_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c1_gputest.log 2>&1; echo "gputest rc=$?" >> gpurun_out/c1_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c1_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dp_hull_kernel -s 1 -c 1 -o gpurun_out/c1_dp python tools/prof_dp.py --entries 4096 --reps 2 > gpurun_out/c1_ncu.log 2>&1
