# self-fed degrees: L2 bulk prefetch of the tile 1 / 2 / 4 beyond the refilled one vs none
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
for k in 1 2 4; do
  echo "## B = prefetch $k" >> gpurun_out/ab_sfpf.txt
  python tools/ab.py $L build/lib_pf$k.so 1e9 6,7,8,12 15 >> gpurun_out/ab_sfpf.txt 2>&1
done
python tools/ab_sustained.py $L build/lib_pf2.so 1e9 8 50 6 >> gpurun_out/ab_sfpf.txt 2>&1
