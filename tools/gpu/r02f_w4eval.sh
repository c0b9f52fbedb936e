timeout 600 ncu --set full --import-source on --clock-control none -k regex:eval_p32 -s 3 -c 1 \
  -o gpurun_out/w4eval python bench.py --workload W4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/w4eval.log 2>&1
