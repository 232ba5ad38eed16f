# 8-tile folds for the product degrees 3, 4 (A/B), then ncu --set full of the m = 3 product kernel at n = 4e9
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab_sustained.py $L build/lib_f3.so 4e9 3 20 6 > gpurun_out/ab_fold34.txt 2>&1
python tools/ab_sustained.py $L build/lib_f3p.so 1e9 4 50 6 >> gpurun_out/ab_fold34.txt 2>&1
python tools/ab_sustained.py $L build/lib_f3.so 1e8 3 300 6 >> gpurun_out/ab_fold34.txt 2>&1
python tools/ab.py $L build/lib_f3p.so 1e9 3,4 15 >> gpurun_out/ab_fold34.txt 2>&1
python tools/prof_target.py 4e9 3 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:power_sums_kernel -c 1 -o gpurun_out/r02c_ps3 python tools/prof_target.py 4e9 3 > gpurun_out/ncu_full.log 2>&1
