# half-tile ring slots for the split degrees (default) vs full-tile slots
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py build/lib_h0.so $L 1e9 6,7,8,10,12 20 > gpurun_out/ab_half.txt 2>&1
python tools/ab.py build/lib_h0.so $L 1e8 6,8,12 30 >> gpurun_out/ab_half.txt 2>&1
python tools/ab_sustained.py build/lib_h0.so $L 1e9 6 50 6 >> gpurun_out/ab_half.txt 2>&1
python tools/ab_sustained.py build/lib_h0.so $L 1e9 8 50 6 >> gpurun_out/ab_half.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > gpurun_out/pytest_half.log 2>&1
