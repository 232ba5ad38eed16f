LSQ_PARITY_OUT=gpurun_out/parity_fs.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "batched or diagnostics" > gpurun_out/pytest_fs.log 2>&1
