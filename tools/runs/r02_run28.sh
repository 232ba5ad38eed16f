python tools/ab_dyn.py 5e7,1e8,2e8,4e8 1,2,3 "0:0:0 8:8:32 4:8:32 4:16:32 16:8:32 8:16:16 4:8:16" 20 > gpurun_out/abdyn2.log 2>&1
