LSQFIT_CUDA_LIB=build/lib_trace.so python tools/ps_trace.py 1,2,3,4,8 1e3,1e6 > gpurun_out/trace3.log 2>&1
