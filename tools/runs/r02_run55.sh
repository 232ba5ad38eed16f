LSQ_PARITY_OUT=gpurun_out/parity_fs3.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "headline or diagnostics" --durations=3 > gpurun_out/pytest_fs3.log 2>&1
