# m = 3 under the power cap: 8-tile folds (f3), self-fed 8 consumers (sf3) vs shipped
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab_sustained.py $L build/lib_f3.so 4e9 3 20 8 > gpurun_out/ab_m3cap.txt 2>&1
python tools/ab_sustained.py $L build/lib_sf3.so 4e9 3 20 8 >> gpurun_out/ab_m3cap.txt 2>&1
python tools/ab.py $L build/lib_sf3.so 1e9 3,4,5 15 >> gpurun_out/ab_m3cap.txt 2>&1
