timeout 900 python -m pytest tests/test_gpu_ordered.py tests/test_reference_suites.py -q -x > gpurun_out/pytest_rows2.log 2>&1
python tools/ordered_perf.py 1e8 16,128,4096,8192,16384,32768,65536,1000000 1,3,8 > gpurun_out/ordered_perf_r02.log 2>&1
