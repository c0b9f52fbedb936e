# A/B: HEAD (ab_old/) vs the working tree on W5 rows, alternating; then ncu of the large-hull
# mode on all-ones rows
for i in 1 2; do
  (cd ab_old && timeout 300 python tools/prof_dp.py --entries 16384 --reps 3) > gpurun_out/ab_old_$i.log 2>&1
  timeout 300 python tools/prof_dp.py --entries 16384 --reps 3 > gpurun_out/ab_new_$i.log 2>&1
done
timeout 600 python tools/prof_dp.py --entries 16384 --reps 2 --ones > gpurun_out/ab_ones.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dp_hull_kernel -s 4 -c 1 \
  -o gpurun_out/big_ones python tools/prof_dp.py --entries 2048 --reps 2 --ones > gpurun_out/big_ones_ncu.log 2>&1
