# ncu --set full of the final high-degree kernels (m = 5 producer-fed, 6 / 8 self-fed with L2 prefetch, 12) at n = 5e8
python tools/prof_target.py 5e8 5,6,8,12 > gpurun_out/plain_hi.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:power_sums_kernel -c 4 -o gpurun_out/r02f_ps_hi python tools/prof_target.py 5e8 5,6,8,12 > gpurun_out/ncu_hi2.log 2>&1
