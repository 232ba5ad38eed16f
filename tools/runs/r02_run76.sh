# final code (solve butterflies): whole GPU suite, smoke, sweep, graph-replayed small fits, bench pair, launch list
LSQ_PARITY_OUT=gpurun_out/parity_final3.jsonl timeout 2400 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/pytest_final3.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final3.log 2>&1
python tools/sweep.py > gpurun_out/sweep_final8.json 2> gpurun_out/sweep_final8.err
./tools/graph_bench 1e3,1e6,1e7,1e8 1,2,3,8 > gpurun_out/graph_final.jsonl 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02e.json 2> gpurun_out/bench_r02e.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_r02e_ref.json 2> gpurun_out/bench_r02e_ref.err
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02e.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_list.log 2>&1
