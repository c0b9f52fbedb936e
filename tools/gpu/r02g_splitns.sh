for i in 1 2; do
  timeout 300 python tools/prof_dp.py --entries 2048 --reps 3 > gpurun_out/ns_main_$i.log 2>&1
  for v in 8 256; do (cd sp_ns$v && timeout 300 python tools/prof_dp.py --entries 2048 --reps 3) > gpurun_out/ns_${v}_$i.log 2>&1; done
done
