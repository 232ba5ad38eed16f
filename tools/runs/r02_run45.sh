L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
LSQFIT_CUDA_LIB=build/lib_tmem.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bound or boundaries" > gpurun_out/pytest_tmem.log 2>&1
python tools/ab.py $L build/lib_tmem.so 1e9 5,6,7,8,10,12 12 > gpurun_out/ab_tmem.log 2>&1
