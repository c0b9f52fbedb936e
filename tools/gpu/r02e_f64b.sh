timeout 900 python tools/prof_f64.py > gpurun_out/f64b.log 2>&1
