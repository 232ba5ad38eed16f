# 16 tiles per fold for m >= 5 vs 8
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
timeout 600 python tools/ab.py $L build/lib_f16.so 1e9 5,6,7,8,10,12 20 > gpurun_out/ab_f16.txt 2>&1
timeout 600 python tools/ab_sustained.py $L build/lib_f16.so 1e9 8 50 6 >> gpurun_out/ab_f16.txt 2>&1
