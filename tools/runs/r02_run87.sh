# final code (warp-specialised m >= 6): whole GPU suite, smoke, sweep, soak, bench pair
LSQ_PARITY_OUT=gpurun_out/parity_final5.jsonl timeout 2400 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/pytest_final5.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final5.log 2>&1
python tools/sweep.py > gpurun_out/sweep_final11.json 2> gpurun_out/sweep_final11.err
python tools/determinism_soak.py 1e8 1000 > gpurun_out/soak_final4.log 2>&1
./tools/graph_bench 1e3,1e6,1e7,1e8 1,2,3,8 > gpurun_out/graph_final3.jsonl 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_r02g_ref.json 2> gpurun_out/bench_r02g_ref.err
