LSQFIT_CUDA_LIB=build/lib_trace.so python tools/ps_trace.py 1,3,8 1e3,1e6,1e8 > gpurun_out/trace2.log 2>&1
python tools/ab_dyn.py 4e9 1,2,3 "0:0:0 8:16:32 4:16:64 8:8:32" 12 > gpurun_out/abdyn4e9.log 2>&1
