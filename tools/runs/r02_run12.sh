L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py build/lib_noprod.so $L 1e9 4,5,6,7,8,9,10,11,12 12 > gpurun_out/ab_prod.log 2>&1
python tools/ab.py build/lib_cl2.so $L 1e9 5,6,7,8,10,12 12 >> gpurun_out/ab_prod.log 2>&1
python tools/ab.py build/lib_cl8.so $L 1e9 5,6,7,8,10,12 12 >> gpurun_out/ab_prod.log 2>&1
LSQ_PARITY_OUT=gpurun_out/parity_full2.jsonl timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_streaming.py tests/test_gpu_fullsize.py tests/test_capi_cpu.py -q -x > gpurun_out/pytest_prod.log 2>&1
