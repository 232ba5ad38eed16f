python tools/ab_dyn.py 5e7,1e8,2e8,4e8 2,3 "0:0:0 2:8:64 4:8:64 4:16:64 8:8:32 8:16:32 4:8:32" 30 > gpurun_out/abdyn.log 2>&1
python tools/ab_dyn.py 1e6,1e7 1,3 "0:0:0 4:8:1 8:2:1" 30 >> gpurun_out/abdyn.log 2>&1
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_target.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.log
