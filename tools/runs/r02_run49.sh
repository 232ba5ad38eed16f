LSQ_PARITY_OUT=gpurun_out/parity_head2.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_head2.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_head2.log 2>&1
