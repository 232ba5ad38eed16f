L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py $L build/lib_cl16b.so 1e9 5,6,7,8,10,12 12 > gpurun_out/ab_shape2.log 2>&1
python tools/ab.py $L build/lib_f16.so 1e9 5,6,7,8,10,12 12 >> gpurun_out/ab_shape2.log 2>&1
python tools/ab.py $L build/lib_loreg.so 1e9 6,7,8 12 >> gpurun_out/ab_shape2.log 2>&1
