L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py build/lib_cw16.so $L 1e9 7,8,9,10 12 > gpurun_out/ab_cw16.log 2>&1
