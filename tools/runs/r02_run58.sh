# per-warp rings (default now) vs the shared-tile ring, + L2 prefetch variants + compute-only probe
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py build/lib_ring0.so $L 1e9 5,6,7,8,10,12 15 > gpurun_out/ab_ring.txt 2>&1
python tools/ab.py $L build/lib_pf2.so 1e9 5,6,7,8 15 > gpurun_out/ab_pf2.txt 2>&1
python tools/ab.py $L build/lib_pf4.so 1e9 5,6,7,8 15 > gpurun_out/ab_pf4.txt 2>&1
python tools/ab.py $L build/lib_probe1.so 1e9 5,6,7,8 15 > gpurun_out/ab_probe1_ring.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/pytest_ring.log 2>&1
