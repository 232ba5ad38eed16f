"""Sustained A/B of two library builds: blocks of K back-to-back launches
(the bench's regime: power-capped clocks), alternating A, B, A, B ...
usage: python tools/ab_sustained.py libA libB n m [K] [blocks]"""
import ctypes as C
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import device as D  # noqa: E402


def load(path):
    L = C.CDLL(path)
    L.lsqfit_cuda_create.argtypes = [C.POINTER(C.c_void_p), C.c_int]
    L.lsqfit_cuda_fit_device.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_uint, C.c_void_p,
                                         C.c_void_p]
    h = C.c_void_p()
    assert L.lsqfit_cuda_create(C.byref(h), 0) == 0
    return L, h


def main():
    n, m = int(float(sys.argv[3])), int(sys.argv[4])
    K = int(sys.argv[5]) if len(sys.argv) > 5 else 50
    blocks = int(sys.argv[6]) if len(sys.argv) > 6 else 4
    xy = D.synth(n, 0, 4, 3, 0.1)
    libs = {"A": load(sys.argv[1]), "B": load(sys.argv[2])}
    out = D.empty_result(xy.device)
    st = torch.cuda.current_stream().cuda_stream
    res = {"A": [], "B": []}
    clk = {"A": [], "B": []}
    samples, stop = [], threading.Event()
    try:  # SM clock samples (NVML, every ~2 ms) to attribute power-capped blocks
        import pynvml as nv
        nv.nvmlInit()
        hdl = nv.nvmlDeviceGetHandleByIndex(0)

        def poll():
            while not stop.is_set():
                samples.append((time.perf_counter(), nv.nvmlDeviceGetClockInfo(hdl, nv.NVML_CLOCK_SM)))
                time.sleep(0.002)
        threading.Thread(target=poll, daemon=True).start()
    except Exception:  # pragma: no cover
        pass
    for b in range(blocks + 1):
        for k in ("A", "B") if b % 2 == 0 else ("B", "A"):
            L, h = libs[k]
            for _ in range(3):
                L.lsqfit_cuda_fit_device(h, xy.data_ptr(), n, m, 1, out.data_ptr(), st)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            for _ in range(K):
                L.lsqfit_cuda_fit_device(h, xy.data_ptr(), n, m, 1, out.data_ptr(), st)
            e1.record()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            if b > 0:
                res[k].append(e0.elapsed_time(e1) / K)
                cs = [c for t, c in samples if t0 <= t <= t1]
                clk[k].append(statistics.median(cs) if cs else None)
    ma, mb = statistics.median(res["A"]), statistics.median(res["B"])
    print(f"sustained m={m} n={n:.0e} K={K}: A {ma:.4f} ms ({16*n/ma/1e6:.0f} GB/s)  "
          f"B {mb:.4f} ms ({16*n/mb/1e6:.0f} GB/s)  B/A {mb/ma:.3f}  A={['%.3f' % v for v in res['A']]} "
          f"B={['%.3f' % v for v in res['B']]}  sm_mhz A={clk['A']} B={clk['B']}", flush=True)
    stop.set()


if __name__ == "__main__":
    main()
