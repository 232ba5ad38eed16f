# m = 4 with product terms: shape variants (dynamic tail, + round-robin deal, the self-fed split shape of m >= 5)
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
for V in d4 g4 sf4; do
  echo "## B = $V" >> gpurun_out/ab_m4.txt
  python tools/ab.py $L build/lib_$V.so 1e9 4 15 >> gpurun_out/ab_m4.txt 2>&1
  python tools/ab.py $L build/lib_$V.so 1e8 4 30 >> gpurun_out/ab_m4.txt 2>&1
  python tools/ab_sustained.py $L build/lib_$V.so 1e9 4 50 6 >> gpurun_out/ab_m4.txt 2>&1
done
