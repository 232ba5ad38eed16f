"""Dev probe: H2D bandwidth from default pinned vs write-combined pinned host
memory (cudaHostAllocWriteCombined: no CPU caching, no snoop on PCIe reads)."""
import ctypes as C
import json
import time
import torch

rt = C.CDLL("libcudart.so")
n_bytes = 8 << 30
dev = torch.empty(n_bytes, dtype=torch.uint8, device="cuda")
out = {}
for label, flags in (("default", 0), ("write_combined", 4), ("portable_mapped", 1 | 2)):
    p = C.c_void_p()
    assert rt.cudaHostAlloc(C.byref(p), C.c_size_t(n_bytes), C.c_uint(flags)) == 0
    C.memset(p, 1, n_bytes)
    best = 0.0
    for r in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        assert rt.cudaMemcpy(C.c_void_p(dev.data_ptr()), p, C.c_size_t(n_bytes), 1) == 0  # H2D
        torch.cuda.synchronize()
        best = max(best, n_bytes / (time.perf_counter() - t0) / 1e9)
    out[label] = round(best, 2)
    rt.cudaFreeHost(p)
print(json.dumps({"h2d_GBps": out}))
