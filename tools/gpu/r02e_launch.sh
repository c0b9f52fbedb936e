# launch lists (our kernels only) of the W5 bench step and of the small configs
K='regex:lcp_hist|row_stats|dp_hull|dp_place|eval_bcast|eval_p32|accumulate|Radix|DeviceRadix'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 60 --csv \
  --log-file gpurun_out/r02e_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/r02e_ncu_launches.log 2>&1
for w in W3 W2; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 60 --csv \
  --log-file gpurun_out/r02e_launches_$w.csv python bench.py --workload $w --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/r02e_ncu_launches_$w.log 2>&1
done
