for i in 1 2 3; do ./tools/cudart_init_probe; ./tools/init_breakdown; python tools/cuinit_probe.py; done > gpurun_out/init2.log 2>&1
