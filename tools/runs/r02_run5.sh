LSQFIT_CUDA_LIB=build/lib_trace.so python tools/ps_trace.py 1,3,8 1e6,1e7,1e8,1e9 > gpurun_out/trace.log 2>&1
python tools/n_sweep.py > gpurun_out/nsweep.log 2>&1
