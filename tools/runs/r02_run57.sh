# probe: compute-only (PROBE 1) and compute+release (PROBE 2) vs the shipped kernel, m = 5..8
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py $L build/lib_probe1.so 1e9 5,6,7,8 15 > gpurun_out/probe1.txt 2>&1
python tools/ab.py $L build/lib_probe2.so 1e9 5,6,7,8 15 > gpurun_out/probe2.txt 2>&1
