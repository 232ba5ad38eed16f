# per-CTA timeline at mid sizes + coarser mid-size tail plans
LSQFIT_CUDA_LIB=build/lib_trace.so python tools/ps_trace.py 2,3,5 1e8,2e8 > gpurun_out/trace_mid.txt 2>&1
python tools/ab_dyn.py 1e8,2e8 2,3,5 "8:16:32 8:32:32 16:16:32 16:8:32 6:16:32 12:16:32 8:24:32" 30 > gpurun_out/ab_mid2.txt 2>&1
