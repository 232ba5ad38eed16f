# products from m = 3 (now default) vs from m = 5 (before): sustained + burst A/B, GPU suite, headline full-size parity
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab_sustained.py build/lib_prod5.so $L 4e9 3 20 6 > gpurun_out/ab_prod3.txt 2>&1
python tools/ab_sustained.py build/lib_prod5.so $L 1e9 4 50 6 >> gpurun_out/ab_prod3.txt 2>&1
python tools/ab_sustained.py build/lib_prod5.so $L 1e8 3 300 6 >> gpurun_out/ab_prod3.txt 2>&1
python tools/ab.py build/lib_prod5.so $L 1e9 3,4 15 >> gpurun_out/ab_prod3.txt 2>&1
python tools/ab.py build/lib_prod5.so $L 1e8 3,4 30 >> gpurun_out/ab_prod3.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/pytest_prod3.log 2>&1
LSQ_PARITY_OUT=gpurun_out/parity_prod3.jsonl timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "headline" --durations=3 >> gpurun_out/pytest_prod3.log 2>&1
