# sustained (power-capped regime) A/B: reference terms (shipped) vs product terms from m = 2
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab_sustained.py $L build/lib_prod2.so 4e9 3 20 6 > gpurun_out/ab_prod_sustained.txt 2>&1
python tools/ab_sustained.py $L build/lib_prod2.so 1e9 4 50 6 >> gpurun_out/ab_prod_sustained.txt 2>&1
python tools/ab_sustained.py $L build/lib_prod2.so 1e8 2 300 6 >> gpurun_out/ab_prod_sustained.txt 2>&1
python tools/ab.py $L build/lib_prod2.so 1e9 2,3,4 15 >> gpurun_out/ab_prod_sustained.txt 2>&1
nvidia-smi --query-gpu=power.limit,clocks.max.sm --format=csv >> gpurun_out/ab_prod_sustained.txt
