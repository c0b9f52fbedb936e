# ptxas scheduling variants of the whole library on W5 rows (prof_dp, 16384 entries)
for i in 1 2; do
  timeout 300 python tools/prof_dp.py --entries 16384 --reps 3 > gpurun_out/fl_main_$i.log 2>&1
  for v in rul8 rul2 aeo rul10; do
    (cd variants/$v && timeout 300 python tools/prof_dp.py --entries 16384 --reps 3) > gpurun_out/fl_${v}_$i.log 2>&1
  done
done
