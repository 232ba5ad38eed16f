L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py build/lib_cw10.so $L 1e9 7,8,10,12 10 > gpurun_out/ab_cw.log 2>&1
python tools/ab.py build/lib_cw8.so $L 1e9 7,8,10,12 10 >> gpurun_out/ab_cw.log 2>&1
