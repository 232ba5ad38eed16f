# m = 4 dynamic tail + round-robin deal: parity tests, sweep
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_streaming.py tests/test_gpu_ordered.py -q -x > gpurun_out/pytest_m4dyn.log 2>&1
python tools/sweep.py > gpurun_out/sweep_final5.json 2> gpurun_out/sweep_final5.err
