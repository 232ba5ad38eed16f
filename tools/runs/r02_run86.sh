# warp-specialised split shape with the L2 prefetch (m = 6..8) vs self-fed (shipped); and without prefetch
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
timeout 600 python tools/ab.py $L build/lib_ws.so 1e9 6,7,8,9,10,12 20 > gpurun_out/ab_ws2.txt 2>&1
timeout 600 python tools/ab.py $L build/lib_ws.so 1e8 6,7,8 30 >> gpurun_out/ab_ws2.txt 2>&1
timeout 600 python tools/ab.py $L build/lib_ws.so 1e6 6,8 40 >> gpurun_out/ab_ws2.txt 2>&1
timeout 600 python tools/ab.py build/lib_wsnp.so build/lib_ws.so 1e9 6,7,8 20 >> gpurun_out/ab_ws2.txt 2>&1
timeout 600 python tools/ab_sustained.py $L build/lib_ws.so 1e9 6 50 6 >> gpurun_out/ab_ws2.txt 2>&1
timeout 600 python tools/ab_sustained.py $L build/lib_ws.so 1e9 7 50 6 >> gpurun_out/ab_ws2.txt 2>&1
timeout 600 python tools/ab_sustained.py $L build/lib_ws.so 1e9 8 50 6 >> gpurun_out/ab_ws2.txt 2>&1
