# TMA-fed batched warp kernel (default 16 warps x 3 slots) vs the LDG kernel; shape variants; batched tests
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab_batched.py build/lib_bt0.so $L 2:1024:1000000 2:4096:250000 8:1024:1000000 3:2048:500000 1:1000:1000000 2:1023:1000000 5:3000:300000 > gpurun_out/ab_bt.txt 2>&1
python tools/ab_batched.py build/lib_bt0.so build/lib_bt86.so 2:1024:1000000 3:2048:500000 8:1024:1000000 >> gpurun_out/ab_bt.txt 2>&1
python tools/ab_batched.py build/lib_bt0.so build/lib_bt124.so 2:1024:1000000 3:2048:500000 8:1024:1000000 >> gpurun_out/ab_bt.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py -q -x > gpurun_out/pytest_bt.log 2>&1
