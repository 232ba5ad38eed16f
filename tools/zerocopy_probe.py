"""Dev probe: can the fused kernel read pinned HOST memory directly over PCIe
(zero-copy, UVA pointer) faster than cudaMemcpy H2D (the e2e path)? Prints
H2D copy GB/s (1 and 2 streams) and the kernel's GB/s on host-mapped input."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1512_08017_b200 import _capi, device as D

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 250_000_000
m = 3
dev = torch.device("cuda", 0)
xy = D.synth(n, 0, 4, 3, 0.1, device=dev)
host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
host.copy_(xy)
torch.cuda.synchronize()
out = {}
dbuf = torch.empty_like(xy)
for rep in range(3):
    t0 = time.perf_counter(); dbuf.copy_(host, non_blocking=True); torch.cuda.synchronize()
    out["h2d_1stream_GBps"] = 16 * n / (time.perf_counter() - t0) / 1e9
s2 = torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = n // 2
    dbuf[:h].copy_(host[:h], non_blocking=True)
    with torch.cuda.stream(s2):
        dbuf[h:].copy_(host[h:], non_blocking=True)
    torch.cuda.synchronize()
    out["h2d_2streams_GBps"] = 16 * n / (time.perf_counter() - t0) / 1e9
ref = D.read_result(D.fit(xy, m))
ctx = _capi.context(0)
res = D.empty_result(dev)
st = torch.cuda.current_stream().cuda_stream
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rc = ctx.fit_device(host.data_ptr(), n, m, _capi.SOLVE, res.data_ptr(), st)
    torch.cuda.synchronize()
    out["zero_copy_kernel_GBps"] = 16 * n / (time.perf_counter() - t0) / 1e9
    out["zero_copy_rc"] = rc
r = D.read_result(res)
out["zero_copy_bitwise_equal_to_device"] = list(r.coeffs[:4]) == list(ref.coeffs[:4])
print(json.dumps(out))
