# final kernel: the whole GPU suite (full-size parity recorded), the secondary sweep, the determinism soak
LSQ_PARITY_OUT=gpurun_out/parity_final.jsonl timeout 2400 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/pytest_final.log 2>&1
python tools/sweep.py > gpurun_out/sweep_final4.json 2> gpurun_out/sweep_final4.err
python tools/determinism_soak.py 1e8 1000 > gpurun_out/soak_final.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1
