timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_streaming.py tests/test_gpu_ordered.py tests/test_capi_cpu.py -q -x > gpurun_out/pytest_m5.log 2>&1
python tools/determinism_soak.py 1e8 1000 > gpurun_out/soak_m5.log 2>&1
python tools/sweep.py > gpurun_out/sweep_final3.json 2> gpurun_out/sweep_final3.err
