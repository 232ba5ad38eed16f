LSQ_PARITY_OUT=gpurun_out/parity_fs2.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "tsqr" > gpurun_out/pytest_fs2.log 2>&1
