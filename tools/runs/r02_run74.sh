# final code: whole GPU suite (full-size parity recorded), sweep, determinism soak, smoke, bench pair
LSQ_PARITY_OUT=gpurun_out/parity_final2.jsonl timeout 2400 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/pytest_final2.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final2.log 2>&1
python tools/sweep.py > gpurun_out/sweep_final7.json 2> gpurun_out/sweep_final7.err
python tools/determinism_soak.py 1e8 1000 > gpurun_out/soak_final2.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_r02d_ref.json 2> gpurun_out/bench_r02d_ref.err
