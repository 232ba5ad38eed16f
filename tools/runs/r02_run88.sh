# warp-specialised shape: L2 prefetch also for m = 9..12 (pf12), prefetch 2 ahead (pf2w) vs shipped
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
timeout 600 python tools/ab.py $L build/lib_pf12.so 1e9 9,10,11,12 20 > gpurun_out/ab_wspf.txt 2>&1
timeout 600 python tools/ab.py $L build/lib_pf2w.so 1e9 6,7,8 20 >> gpurun_out/ab_wspf.txt 2>&1
timeout 600 python tools/ab_sustained.py $L build/lib_pf12.so 1e9 10 40 6 >> gpurun_out/ab_wspf.txt 2>&1
