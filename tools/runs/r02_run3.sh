nvidia-smi -q | grep -i -E "persistence|Addressing|BAR1" -A2 | head -20 > gpurun_out/cuinit.log
for i in 1 2 3; do python tools/cuinit_probe.py; done >> gpurun_out/cuinit.log 2>&1
