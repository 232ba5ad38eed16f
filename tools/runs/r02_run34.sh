L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py $L build/lib_v1.so 1e9 5 16 > gpurun_out/ab_m45.log 2>&1
python tools/ab.py $L build/lib_v2.so 1e9 4 16 >> gpurun_out/ab_m45.log 2>&1
python tools/ab.py $L build/lib_v3.so 1e9 4 16 >> gpurun_out/ab_m45.log 2>&1
python tools/ab.py $L build/lib_v1.so 1e8 5 30 >> gpurun_out/ab_m45.log 2>&1
python tools/ab.py $L build/lib_v2.so 1e8 4 30 >> gpurun_out/ab_m45.log 2>&1
python tools/ab.py $L build/lib_v3.so 1e8 4 30 >> gpurun_out/ab_m45.log 2>&1
