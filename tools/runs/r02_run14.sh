L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py build/lib_m56split.so $L 1e9 5,6 12 > gpurun_out/ab_prod3.log 2>&1
python tools/ab.py build/lib_m6split.so $L 1e9 6 12 >> gpurun_out/ab_prod3.log 2>&1
python tools/ab.py build/lib_cl16.so $L 1e9 5,6 12 >> gpurun_out/ab_prod3.log 2>&1
