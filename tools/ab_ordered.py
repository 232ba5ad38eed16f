"""A/B of the reference-order (bit-exact) slot kernels: the cp.async row
kernel (thread per chunk) switched on / off through the dev hook
lsqfit_debug_set_ordered_rows_min; both must give the same bits.
usage: python tools/ab_ordered.py [n] [chunks,..] [m,..]"""
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import _capi, device as D  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
chunk_list = [int(float(v)) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2**14, 2**15, 2**16, 2**18]
degs = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 3, 8, 12]
hook = _capi.lib().lsqfit_debug_set_ordered_rows_min
hook.argtypes = [C.c_int]
xy = D.synth(n, 0, 4, 3, 0.1)
out = D.empty_result("cuda")
for m in degs:
    for c in chunk_list:
        rec = {"n": n, "m": m, "chunks": c}
        for label, setting in (("rows_kernel", 1), ("round1_kernels", 2**31 - 1)):
            hook(setting)
            ts = []
            for r in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                D.fit_ordered(xy, m, c, out=out)
                e1.record()
                torch.cuda.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1))
            res = D.read_result(out)
            rec[label] = {"ms": round(statistics.median(ts), 3),
                          "coeffs_hex": [float(v).hex() for v in res.coeffs[: m + 1]],
                          "s_hex": [float(v).hex() for v in res.s[: 2 * m + 1]]}
        hook(0)
        rec["bit_identical"] = (rec["rows_kernel"]["coeffs_hex"] == rec["round1_kernels"]["coeffs_hex"]
                                and rec["rows_kernel"]["s_hex"] == rec["round1_kernels"]["s_hex"])
        print(json.dumps({k: (v if not isinstance(v, dict) else v["ms"]) for k, v in rec.items()}), flush=True)
