L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py $L build/lib_lock.so 1e9 5,6,7,8,10,12 12 > gpurun_out/ab_lock.log 2>&1
