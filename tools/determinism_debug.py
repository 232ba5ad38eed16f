"""Which fields differ between repeated launches (determinism soak triage)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1512_08017_b200 import _capi, device as D  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
launches = int(sys.argv[2]) if len(sys.argv) > 2 else 200
degs = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [5, 8]
xy = D.synth(n, 0, 4, 3, 0.1)
B = _capi.RESULT_BYTES
for m in degs:
    outs = torch.empty(launches * B, dtype=torch.uint8, device="cuda")
    for i in range(launches):
        D.fit(xy, m, out=outs[i * B:(i + 1) * B])
    torch.cuda.synchronize()
    host = outs.cpu().numpy().reshape(launches, B)
    recs = [_capi.Result.from_buffer_copy(host[i].tobytes()) for i in range(launches)]
    s0 = np.array(recs[0].s[: 2 * m + 1])
    nd = 0
    for i, r in enumerate(recs[1:], 1):
        s = np.array(r.s[: 2 * m + 1])
        t = np.array(r.t[: m + 1])
        if not (np.array_equal(s, s0) and np.array_equal(t, np.array(recs[0].t[: m + 1]))):
            nd += 1
            if nd <= 3:
                ds = np.nonzero(s != s0)[0]
                print(f"m={m} launch {i}: s differs at {ds.tolist()} rel {np.max(np.abs(s - s0) / np.abs(s0)):.3e}; "
                      f"hi equal {np.array_equal(np.array(r.part_hi[:3*m+1]), np.array(recs[0].part_hi[:3*m+1]))}",
                      flush=True)
    print(f"m={m}: {nd} of {launches - 1} launches differ from the first", flush=True)
