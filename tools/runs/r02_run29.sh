python tools/determinism_soak.py 4e9 300 > gpurun_out/soak_4e9.log 2>&1
python tools/determinism_soak.py 1e8 3000 > gpurun_out/soak_1e8.log 2>&1
python tools/determinism_soak.py 1e6 20000 > gpurun_out/soak_1e6.log 2>&1
