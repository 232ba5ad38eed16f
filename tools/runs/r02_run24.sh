L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py $L build/lib_inl.so 1e6 1,3,5,8,12 40 > gpurun_out/ab_inl.log 2>&1
python tools/ab.py $L build/lib_inl.so 1e8 1,3,8 20 >> gpurun_out/ab_inl.log 2>&1
LSQFIT_CUDA_LIB=build/lib_trace_inl.so python tools/ps_trace.py 1,3,8 1e3 > gpurun_out/trace_inl.log 2>&1
