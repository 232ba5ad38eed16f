# mid-size dynamic-tail plans: guided chunk sizes ending at 2-8 tiles (den:chunk:min, runtime hook)
python tools/ab_dyn.py 5e7,1e8,2e8 2,3,4,5 "8:16:32 4:4:32 4:2:32 8:4:32 8:2:32 4:8:32 6:4:32" 30 > gpurun_out/ab_mid.txt 2>&1
