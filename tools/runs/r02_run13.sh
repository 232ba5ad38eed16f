L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py build/lib_nosplit.so $L 1e9 7,8,10,12 12 > gpurun_out/ab_prod2.log 2>&1
python tools/ab.py build/lib_fold4.so $L 1e9 7,8,10,12 12 >> gpurun_out/ab_prod2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:power_sums_kernel -o gpurun_out/ps_prod python tools/prof_target.py 5e8 5,6,8 > gpurun_out/ncu_prod.log 2>&1
