L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py $L build/lib_p16s.so 1e9 7,8,10,12 12 > gpurun_out/ab_p16s.log 2>&1
python tools/ab.py $L build/lib_p16s_f4.so 1e9 7,8,10,12 12 >> gpurun_out/ab_p16s.log 2>&1
