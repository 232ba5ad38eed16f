"""Dev probe: split CUDA initialisation into cuInit and primary-context creation."""
import ctypes, json, time
t0 = time.perf_counter()
cu = ctypes.CDLL("libcuda.so.1")
t1 = time.perf_counter()
r1 = cu.cuInit(0)
t2 = time.perf_counter()
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
ctx = ctypes.c_void_p()
r2 = cu.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev)
t3 = time.perf_counter()
r3 = cu.cuCtxSetCurrent(ctx)
free, total = ctypes.c_size_t(), ctypes.c_size_t()
cu.cuMemGetInfo_v2(ctypes.byref(free), ctypes.byref(total))
t4 = time.perf_counter()
print(json.dumps({"dlopen_ms": (t1 - t0) * 1e3, "cuInit_ms": (t2 - t1) * 1e3, "ctx_retain_ms": (t3 - t2) * 1e3,
                  "set_current_meminfo_ms": (t4 - t3) * 1e3, "rc": [r1, r2, r3]}))
