for i in 1 2 3; do ./tools/init_breakdown; done > gpurun_out/init.log 2>&1
for i in 1 2; do CUDA_MODULE_LOADING=EAGER ./tools/init_breakdown; done >> gpurun_out/init.log 2>&1
for i in 1 2; do oracle/_ref/acceptance_on_b200 | head -2; done >> gpurun_out/init.log 2>&1
python tools/zerocopy_probe.py 2.5e8 > gpurun_out/zerocopy.log 2>&1
