python tools/ab.py build/lib_p16s.so build/lib_p16s_m5.so 1e9 5,6 12 > gpurun_out/ab_p16s_m56.log 2>&1
python tools/ab.py build/lib_p16s.so build/lib_p16s_m6.so 1e9 6 12 >> gpurun_out/ab_p16s_m56.log 2>&1
python tools/ab.py build/lib_p16s.so build/lib_p16s_m5.so 1e8 5,6,7,8 12 >> gpurun_out/ab_p16s_m56.log 2>&1
