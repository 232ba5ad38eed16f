python tools/graph_time.py 1e3,1e6,1e7,1e8 1,2,3,8 > gpurun_out/graph_time.log 2>&1
python tools/ab_dyn.py 1e8 2,3 "0:0:0:1 8:16:32:1 2:8:128:1" 20 >> gpurun_out/graph_time.log 2>&1
