timeout 900 python -m pytest tests/test_gpu_ordered.py -q -x > gpurun_out/pytest_ovl.log 2>&1
python tools/ordered_perf.py 1e8 16,128,1024,4096 1,3,8,12 > gpurun_out/ord_new.log 2>&1
