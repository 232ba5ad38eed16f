python tools/ab_dyn.py 1e3,1e6,1e7,1e8 1,3,8 "0:0:0:0 0:0:0:1" 30 > gpurun_out/abpdl.log 2>&1
python tools/ab_dyn.py 1e8,1e9 2,3 "0:0:0:1 8:16:32:1" 20 >> gpurun_out/abpdl.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_streaming.py -q -x > gpurun_out/pytest_quick.log 2>&1
