L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py build/lib_prev2.so $L 1e9 7,8,10,12 12 > gpurun_out/ab_pend.log 2>&1
