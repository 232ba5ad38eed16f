"""A/B timing of two builds of the C-ABI library in one process: launches
alternate A, B, A, B ... on the same resident data so clocks / power state
affect both equally. usage: python tools/ab.py libA.so libB.so n m [reps]"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import device as D, _capi  # noqa: E402


def load(path):
    L = C.CDLL(path)
    L.lsqfit_cuda_create.argtypes = [C.POINTER(C.c_void_p), C.c_int]
    L.lsqfit_cuda_fit_device.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_uint, C.c_void_p,
                                         C.c_void_p]
    h = C.c_void_p()
    assert L.lsqfit_cuda_create(C.byref(h), 0) == 0
    return L, h


def main():
    a, b = sys.argv[1], sys.argv[2]
    n = int(float(sys.argv[3]))
    degs = [int(v) for v in sys.argv[4].split(",")]
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 30
    xy = D.synth(n, 0, 4, 3, 0.1)
    libs = {"A": load(a), "B": load(b)}
    outs = {k: D.empty_result(xy.device) for k in libs}
    st = torch.cuda.current_stream().cuda_stream
    for m in degs:
        ts = {"A": [], "B": []}
        for r in range(reps + 3):
            for k, (L, h) in (list(libs.items()) if r % 2 == 0 else list(libs.items())[::-1]):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                L.lsqfit_cuda_fit_device(h, xy.data_ptr(), n, m, 1, outs[k].data_ptr(), st)
                e1.record()
                torch.cuda.synchronize()
                if r >= 3:
                    ts[k].append(e0.elapsed_time(e1))
        ra, rb = D.read_result(outs["A"]), D.read_result(outs["B"])
        same = list(ra.coeffs[: m + 1]) == list(rb.coeffs[: m + 1])
        ma, mb = statistics.median(ts["A"]), statistics.median(ts["B"])
        print(f"m={m:2d} n={n:.0e}  A {ma:8.4f} ms ({16*n/ma/1e6:6.0f} GB/s)   B {mb:8.4f} ms ({16*n/mb/1e6:6.0f} GB/s)"
              f"   B/A {mb/ma:6.3f}  coeffs_equal={same} status={ra.status},{rb.status}", flush=True)
    _ = _capi


if __name__ == "__main__":
    main()
