L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py $L build/lib_prod2.so 1e8 2,3 30 > gpurun_out/ab_prod23.log 2>&1
python tools/ab.py $L build/lib_prod2.so 1e9 2,3 12 >> gpurun_out/ab_prod23.log 2>&1
python tools/ab_sustained.py $L build/lib_prod2.so 4e9 3 20 6 >> gpurun_out/ab_prod23.log 2>&1
