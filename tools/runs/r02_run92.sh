# last check of the committed build: whole GPU suite, smoke, bench
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_last2.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/pytest_last2.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_last.json 2> gpurun_out/bench_last.err
