LSQ_PARITY_OUT=gpurun_out/parity_full3.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu2.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python tools/sweep.py > gpurun_out/sweep.json 2> gpurun_out/sweep.err
