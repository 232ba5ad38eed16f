L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py build/lib_rs00.so $L 1e6 7,8,12 40 > gpurun_out/ab_rs2.log 2>&1
python tools/ab.py build/lib_rs00.so $L 1e9 7,8,12 10 >> gpurun_out/ab_rs2.log 2>&1
python tools/ab.py build/lib_rs0.so $L 1e9 7,8,12 10 >> gpurun_out/ab_rs2.log 2>&1
python tools/ab.py build/lib_prev.so build/lib_rs00.so 1e9 7,8,12 10 >> gpurun_out/ab_rs2.log 2>&1
