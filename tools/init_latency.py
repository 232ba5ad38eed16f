"""Dev probe: wall time of the first fit_normal in a fresh process (CUDA init,
module load, context creation) — the reference's acceptance harness requires
the degree-1 Table I fit < 1 s end to end (acceptance.cpp:125-140)."""
import os, sys, time
t0 = time.perf_counter()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1512_08017_b200 import lsqfit as L
t1 = time.perf_counter()
T1 = [(39.206, 751.912), (29.74, 567.121), (21.31, 403.746), (12.087, 221.738), (1.812, 18.8418), (0.001, 1.88672)]
rep = L.fit_normal(L.Dataset(T1), 1)
t2 = time.perf_counter()
rep = L.fit_normal(L.Dataset(T1), 1)
t3 = time.perf_counter()
print({"import_s": t1 - t0, "first_fit_s": t2 - t1, "second_fit_ms": (t3 - t2) * 1e3, "coeffs": rep.polynomial.coefficients()})
