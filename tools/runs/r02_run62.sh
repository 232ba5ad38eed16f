# bench pair on the product-term m = 3 kernel + launch list
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_r02c_ref.json 2> gpurun_out/bench_r02c_ref.err
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02c.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_list.log 2>&1
