LSQ_PARITY_OUT=gpurun_out/parity_fs4.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "diagnostics" --durations=3 > gpurun_out/pytest_fs4.log 2>&1
