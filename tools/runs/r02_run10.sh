./tools/graph_bench 1e3,1e6,1e7,1e8 1,2,3,8 50 > gpurun_out/graph_bench.log 2>&1
