set -x
python tools/measure_ceilings.py gpurun_out/measured_ceilings.json > gpurun_out/ceil.log 2>&1
cp gpurun_out/measured_ceilings.json profiles/measured_ceilings.json
LSQ_PARITY_OUT=gpurun_out/parity_full.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
