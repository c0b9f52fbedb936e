# final measurement after the one-pass step (r02i)
T=r02i
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench_w5.json 2> gpurun_out/${T}_bench_w5.err
V=gpurun_out/${T}_bench_variants.jsonl
: > $V
timeout 600 python bench.py --entries 2048 --no-cpu-baseline --no-e2e >> $V 2>> gpurun_out/${T}_var.err
timeout 900 python bench.py --weights f64 --no-cpu-baseline >> $V 2>> gpurun_out/${T}_var.err
timeout 900 python bench.py --dp-hist ones --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $V 2>> gpurun_out/${T}_var.err
timeout 900 python bench.py --dp-hist accum --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $V 2>> gpurun_out/${T}_var.err
for w in W2 W3 W4; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e >> $V 2>> gpurun_out/${T}_var.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"lcp_hist|row_stats|dp_hull|dp_place|eval_bcast|eval_p32|accumulate" -c 80 --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/${T}_ncu_launches.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:"lcp_hist|row_stats|dp_hull|dp_place|eval_bcast" -s 21 -c 7 -o gpurun_out/${T}_full \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_full.log 2>&1
