for i in 1 2 3; do ./tools/init_breakdown; done > gpurun_out/init3.log 2>&1
for i in 1 2; do ./tools/cudart_init_probe; oracle/_ref/acceptance_on_b200 | head -2; done >> gpurun_out/init3.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not fullsize" > gpurun_out/pytest_lazy.log 2>&1
