timeout 900 python -m pytest tests/test_gpu_ordered.py -q -x > gpurun_out/pytest_rows.log 2>&1
python tools/ab_ordered.py 1e8 4096,8192,16384,32768,65536,262144 1,3,8,12 > gpurun_out/ab_rows.log 2>&1
