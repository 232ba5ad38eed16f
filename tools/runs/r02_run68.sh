# m = 5 producer-fed: parity tests + sweep
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_streaming.py tests/test_gpu_sharded.py -q -x > gpurun_out/pytest_m5pf.log 2>&1
python tools/sweep.py > gpurun_out/sweep_final6.json 2> gpurun_out/sweep_final6.err
