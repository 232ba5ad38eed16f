nproc; free -g; lscpu | head -20; nvidia-smi --query-gpu=name,power.limit,clocks.max.sm --format=csv
python - <<'PY'
import time, numpy as np, oracle
oracle.build()
print("threads", oracle.max_threads())
n=250_000_000
t=time.time(); xy=oracle.synth(n,0,4,3,0.1); print("synth", n/(time.time()-t))
t=time.time(); r=oracle.exact_sums(xy,3); print("exact m3", n/(time.time()-t))
t=time.time(); r=oracle.exact_sums(xy[:50_000_000],8); print("exact m8", 5e7/(time.time()-t))
ds=oracle.RefDataset(xy)
t=time.time(); ds.accumulate_parallel(3,128); print("refpar", n/(time.time()-t))
t=time.time(); ds.accumulate_parallel(3,128); print("refpar", n/(time.time()-t))
PY
