# source-level ncu capture of the int32 hull kernel (rep 1 of prof_dp.py; launches per rep:
# dp_hull_kernel<int,K,int> then the (empty-list) int64 instantiation)
ENT=${ENT:-4096}
TAG=${TAG:-dp}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dp_hull_kernel -s 2 -c 1 \
  -o gpurun_out/${TAG} python tools/prof_dp.py --entries $ENT --reps 2 > gpurun_out/${TAG}_ncu.log 2>&1
