LSQ_PARITY_OUT=gpurun_out/parity_head3.jsonl timeout 2700 python -m pytest tests -m gpu -q -rs --durations=8 > gpurun_out/pytest_head3.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_head3.log 2>&1
