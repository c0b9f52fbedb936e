timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"long long" -s 1 -c 1 \
  -o gpurun_out/i64 python tools/prof_dp.py --entries 4096 --reps 2 --dense-n 120000 180000 > gpurun_out/i64_ncu.log 2>&1
