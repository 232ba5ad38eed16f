"""A/B of the diagnostics pass between two library builds (alternating
launches on the same resident data). usage: python tools/ab_diag.py libA libB n m[,m..] [reps]"""
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
    L.lsqfit_cuda_diagnostics_device.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p,
                                                 C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
    h = C.c_void_p()
    assert L.lsqfit_cuda_create(C.byref(h), 0) == 0
    return L, h


def main():
    n = int(float(sys.argv[3]))
    degs = [int(v) for v in sys.argv[4].split(",")]
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 20
    xy = D.synth(n, 0, 4, 3, 0.1)
    res = torch.empty(n, dtype=torch.float64, device="cuda")
    libs = {"A": load(sys.argv[1]), "B": load(sys.argv[2])}
    outs = {k: torch.zeros(_capi.DIAG_BYTES, dtype=torch.uint8, device="cuda") for k in libs}
    st = torch.cuda.current_stream().cuda_stream
    for m in degs:
        fr = D.fit(xy, m)
        coeffs = fr[_capi.Result.coeffs.offset:_capi.Result.coeffs.offset + 8 * (m + 1)]
        for with_res in (False, True):
            ts = {"A": [], "B": []}
            for r in range(reps + 3):
                order = list(libs.items()) if r % 2 == 0 else list(libs.items())[::-1]
                for k, (L, h) in order:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    L.lsqfit_cuda_diagnostics_device(h, xy.data_ptr(), n, m, coeffs.data_ptr(), None,
                                                     float("nan"), res.data_ptr() if with_res else None,
                                                     outs[k].data_ptr(), st)
                    e1.record()
                    torch.cuda.synchronize()
                    if r >= 3:
                        ts[k].append(e0.elapsed_time(e1))
            same = bytes(outs["A"].cpu().numpy()) == bytes(outs["B"].cpu().numpy())
            ma, mb = statistics.median(ts["A"]), statistics.median(ts["B"])
            b = (24 if with_res else 16) * n
            print(f"m={m:2d} residuals={int(with_res)}  A {ma:7.3f} ms ({b/ma/1e6:5.0f} GB/s)  "
                  f"B {mb:7.3f} ms ({b/mb/1e6:5.0f} GB/s)  B/A {mb/ma:5.3f}  same={same}", flush=True)


if __name__ == "__main__":
    main()
