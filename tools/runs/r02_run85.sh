# warp-specialised split shape (setmaxnreg: 8 consumers at 240 regs + 4-warp producer group) vs self-fed
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
timeout 600 python tools/ab.py $L build/lib_ws.so 1e9 6,7,8,9,10,11,12 20 > gpurun_out/ab_ws.txt 2>&1
timeout 600 python tools/ab.py $L build/lib_ws.so 1e8 6,8,12 30 >> gpurun_out/ab_ws.txt 2>&1
timeout 600 python tools/ab.py $L build/lib_ws.so 1e3,1e6 6 30 >> gpurun_out/ab_ws.txt 2>&1
timeout 600 python tools/ab_sustained.py $L build/lib_ws.so 1e9 6 50 6 >> gpurun_out/ab_ws.txt 2>&1
timeout 600 python tools/ab_sustained.py $L build/lib_ws.so 1e9 8 50 6 >> gpurun_out/ab_ws.txt 2>&1
