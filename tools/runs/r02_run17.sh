L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_streaming.py -q -x > gpurun_out/pytest_rs.log 2>&1
./tools/graph_bench 1e3,1e6,1e8 1,2,3,5,8 50 > gpurun_out/graph_bench3.log 2>&1
python tools/ab.py build/lib_prev.so $L 1e6 1,2,3,8 40 > gpurun_out/ab_rs.log 2>&1
python tools/ab.py build/lib_prev.so $L 1e8 1,2,3,5,8 20 >> gpurun_out/ab_rs.log 2>&1
python tools/ab.py build/lib_prev.so $L 1e9 3,6,8,12 10 >> gpurun_out/ab_rs.log 2>&1
LSQFIT_CUDA_LIB=build/lib_trace.so python tools/ps_trace.py 1,3,8 1e3,1e6,1e8 > gpurun_out/trace4.log 2>&1
