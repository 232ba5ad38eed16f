# L2 prefetch 1 tile ahead for the self-fed m = 6, 7: longer A/B
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py $L build/lib_pf1.so 1e9 6,7,8 40 > gpurun_out/ab_sfpf1.txt 2>&1
python tools/ab_sustained.py $L build/lib_pf1.so 1e9 6 50 8 >> gpurun_out/ab_sfpf1.txt 2>&1
python tools/ab_sustained.py $L build/lib_pf1.so 1e9 7 50 8 >> gpurun_out/ab_sfpf1.txt 2>&1
python tools/ab.py $L build/lib_pf1.so 1e8 6,7 40 >> gpurun_out/ab_sfpf1.txt 2>&1
