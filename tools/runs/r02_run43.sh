L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab_batched.py $L build/lib_bu2.so 2:1024:1000000 3:1024:1000000 2:4096:250000 > gpurun_out/ab_bu.log 2>&1
python tools/ab_batched.py $L build/lib_bu4.so 2:1024:1000000 3:1024:1000000 2:4096:250000 >> gpurun_out/ab_bu.log 2>&1
