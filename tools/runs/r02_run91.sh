# batched warp kernel: cross-curve prefetch of the next curve's first chunk (XPF, default build) vs none; XPF capped at 64 regs
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab_batched.py build/lib_bx0.so $L 2:1024:1000000 2:4096:250000 3:2048:500000 1:1000:1000000 > gpurun_out/ab_bx.txt 2>&1
python tools/ab_batched.py build/lib_bx0.so build/lib_bx4.so 2:1024:1000000 2:4096:250000 3:2048:500000 >> gpurun_out/ab_bx.txt 2>&1
