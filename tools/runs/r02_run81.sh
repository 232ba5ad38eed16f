timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_streaming.py -q -x > gpurun_out/pytest_pf.log 2>&1
python tools/sweep.py > gpurun_out/sweep_final9.json 2> gpurun_out/sweep_final9.err
