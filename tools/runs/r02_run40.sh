python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_r02b_ref.json 2> gpurun_out/bench_r02b_ref.err
