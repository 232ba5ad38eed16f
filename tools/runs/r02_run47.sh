python tools/ab_ordered.py 1e8 8192,16384,32768,65536 1,3,8,12 > gpurun_out/ab_rows2.log 2>&1
LSQFIT_CUDA_LIB=build/lib_rows3.so python tools/ab_ordered.py 1e8 8192,16384,32768,65536 1,3,8,12 > gpurun_out/ab_rows3.log 2>&1
