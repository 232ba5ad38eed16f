# inline vs noinline solve: epilogue trace + A/B at small and mid sizes
LSQFIT_CUDA_LIB=build/lib_trace.so python tools/ps_trace.py 1,2,3,5,8 1e3,1e6,1e8 > gpurun_out/trace_solve.txt 2>&1
echo "# inline" >> gpurun_out/trace_solve.txt
LSQFIT_CUDA_LIB=build/lib_trace_inl.so python tools/ps_trace.py 1,2,3,5,8 1e3,1e6,1e8 >> gpurun_out/trace_solve.txt 2>&1
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py $L build/lib_inl.so 1e6 1,2,3,5,8 40 > gpurun_out/ab_inl.txt 2>&1
python tools/ab.py $L build/lib_inl.so 1e8 2,3,5 30 >> gpurun_out/ab_inl.txt 2>&1
