# warp solve: butterflies over the first P2 >= DIM lanes + broadcast (default) vs 5-level butterflies
L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py build/lib_old.so $L 1e3 1,2,3,5,8,12 60 > gpurun_out/ab_solve.txt 2>&1
python tools/ab.py build/lib_old.so $L 1e6 1,2,3 60 >> gpurun_out/ab_solve.txt 2>&1
./tools/graph_bench > gpurun_out/graph_new.jsonl 2>&1
LSQFIT_CUDA_LIB=build/lib_old.so ./tools/graph_bench > gpurun_out/graph_old.jsonl 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_streaming.py tests/test_gpu_sharded.py tests/test_gpu_fuzz.py -q -x > gpurun_out/pytest_solve.log 2>&1
