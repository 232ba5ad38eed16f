# m = 5, 6 in the producer-fed product shape (7 consumers + producer, no split) vs the self-fed split shape
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
for V in pf5 pf5d pf6d; do
  echo "## B = $V" >> gpurun_out/ab_pf56.txt
  python tools/ab.py $L build/lib_$V.so 1e9 5,6 15 >> gpurun_out/ab_pf56.txt 2>&1
  python tools/ab.py $L build/lib_$V.so 1e8 5,6 30 >> gpurun_out/ab_pf56.txt 2>&1
  python tools/ab_sustained.py $L build/lib_$V.so 1e9 5 50 6 >> gpurun_out/ab_pf56.txt 2>&1
done
python tools/ab_sustained.py $L build/lib_pf6d.so 1e9 6 50 6 >> gpurun_out/ab_pf56.txt 2>&1
