"""Minimal ncu target: one launch of the fused fit kernel per listed degree."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1512_08017_b200 import device as D
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
degs = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [3, 8]
xy = D.synth(n, 0, 4, 3, 0.1)
for m in degs:
    r = D.read_result(D.fit(xy, m))
    torch.cuda.synchronize()
    print(m, r.status, list(r.coeffs[:2]))
