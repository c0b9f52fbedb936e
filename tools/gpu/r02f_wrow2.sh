timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/wr2_gputest.log 2>&1
V=gpurun_out/wr2_variants.jsonl; : > $V
timeout 900 python bench.py --weights f64 --no-cpu-baseline >> $V 2>> gpurun_out/wr2.err
timeout 900 python bench.py --dp-hist accum --steps 3 --warmup 3 --no-cpu-baseline --no-e2e >> $V 2>> gpurun_out/wr2.err
