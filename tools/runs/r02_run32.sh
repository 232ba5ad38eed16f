L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py $L build/lib_rs11.so 1e6 6,8,12 40 > gpurun_out/ab_rs11.log 2>&1
python tools/ab.py $L build/lib_rs11.so 1e9 6,8,12 10 >> gpurun_out/ab_rs11.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_streaming.py tests/test_capi_cpu.py -q -x > gpurun_out/pytest_p16.log 2>&1
python tools/determinism_soak.py 2e8 500 > gpurun_out/soak_p16.log 2>&1
