# point-major product columns (LSQ_POINT_MAJOR=1) vs the shipped column-major trees, m = 5..12
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py $L build/lib_pm.so 1e9 5,6,7,8,9,10,11,12 15 > gpurun_out/ab_pm.txt 2>&1
python tools/ab.py $L build/lib_pm.so 1e8 5,6,8,12 30 >> gpurun_out/ab_pm.txt 2>&1
