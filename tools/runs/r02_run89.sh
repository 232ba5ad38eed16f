# warp-specialised shape also for m = 3..5 (8 consumers at 232 + producer group at 40, dynamic tail kept) vs shipped (7 consumers + producer warp)
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
timeout 600 python tools/ab_sustained.py $L build/lib_ws3.so 4e9 3 20 8 > gpurun_out/ab_ws3.txt 2>&1
timeout 600 python tools/ab.py $L build/lib_ws3.so 1e9 3,4,5 20 >> gpurun_out/ab_ws3.txt 2>&1
timeout 600 python tools/ab.py $L build/lib_ws3.so 1e8 3,4,5 30 >> gpurun_out/ab_ws3.txt 2>&1
timeout 600 python tools/ab.py $L build/lib_ws3.so 1e6 3 40 >> gpurun_out/ab_ws3.txt 2>&1
timeout 600 python tools/ab_sustained.py $L build/lib_ws3.so 1e9 5 50 6 >> gpurun_out/ab_ws3.txt 2>&1
