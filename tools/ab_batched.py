"""A/B of two library builds on the batched warp-per-curve kernel (C4-like
configs), alternating blocks of back-to-back launches; also checks that both
builds give bit-identical coefficients and statuses.
usage: python tools/ab_batched.py libA.so libB.so [m:ppc:curves ...]"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import device as D  # noqa: E402


def load(path):
    L = C.CDLL(path)
    L.lsqfit_cuda_create.argtypes = [C.POINTER(C.c_void_p), C.c_int]
    L.lsqfit_cuda_fit_batched_device.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_int,
                                                 C.c_void_p, C.c_void_p, C.c_void_p]
    h = C.c_void_p()
    assert L.lsqfit_cuda_create(C.byref(h), 0) == 0
    return L, h


libs = {"A": load(sys.argv[1]), "B": load(sys.argv[2])}
cases = sys.argv[3:] or ["2:1024:1000000", "2:4096:250000", "8:1024:1000000", "3:2048:500000"]
st = torch.cuda.current_stream().cuda_stream
for case in cases:
    m, ppc, curves = (int(float(v)) for v in case.split(":"))
    xy = D.synth_batched(curves, ppc, 5, min(m, 2), 0.1)
    outs = {k: (torch.empty((curves, m + 1), dtype=torch.float64, device="cuda"),
                torch.empty(curves, dtype=torch.int32, device="cuda")) for k in libs}
    res = {"A": [], "B": []}
    K = 20
    for b in range(7):
        for k in ("A", "B") if b % 2 == 0 else ("B", "A"):
            L, h = libs[k]
            c, s = outs[k]
            call = lambda: L.lsqfit_cuda_fit_batched_device(h, xy.data_ptr(), curves, ppc, m, c.data_ptr(),
                                                            s.data_ptr(), st)
            for _ in range(2):
                assert call() == 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(K):
                call()
            e1.record()
            torch.cuda.synchronize()
            if b > 0:
                res[k].append(e0.elapsed_time(e1) / K)
    same = torch.equal(outs["A"][0].view(torch.int64), outs["B"][0].view(torch.int64)) and \
        torch.equal(outs["A"][1], outs["B"][1])
    ma, mb = statistics.median(res["A"]), statistics.median(res["B"])
    gb = 16 * curves * ppc / 1e6
    print(f"batched m={m} ppc={ppc} curves={curves}: A {ma:.4f} ms ({gb/ma:.0f} GB/s)  B {mb:.4f} ms "
          f"({gb/mb:.0f} GB/s)  B/A {mb/ma:.3f}  bit-identical={same}", flush=True)
    del xy, outs
    torch.cuda.empty_cache()
