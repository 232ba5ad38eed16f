"""Dev probe: PCIe host->device read ceilings on this box.
(a) one cudaMemcpyAsync of a pinned buffer, (b) the same split over 2/4
streams, (c) the fused kernel reading the pinned buffer in place (zero-copy:
cp.async.bulk straight from mapped host memory), (d) fit_host (staged)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import _capi, device as D  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 250_000_000
ctx = _capi.context(0)
xy_dev = D.synth(n, 0, 4, 3, 0.1)
pinned = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
pinned.copy_(xy_dev)
dst = torch.empty_like(xy_dev)
res = {"n": n, "bytes": 16 * n}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 16 * n / min(ts) / 1e9


res["memcpy_1stream_GBps"] = timed(lambda: dst.copy_(pinned, non_blocking=True))
for k in (2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    parts_src = pinned.chunk(k)
    parts_dst = dst.chunk(k)

    def split():
        cur = torch.cuda.current_stream()
        for s, a, b in zip(streams, parts_src, parts_dst):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                b.copy_(a, non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
    res[f"memcpy_{k}streams_GBps"] = timed(split)

out = D.empty_result("cuda")
ref = D.read_result(D.fit(xy_dev, 3, out=D.empty_result("cuda")))
try:
    stream = torch.cuda.current_stream().cuda_stream
    res["zero_copy_kernel_GBps"] = timed(
        lambda: ctx.fit_device(pinned.data_ptr(), n, 3, _capi.SOLVE, out.data_ptr(), stream))
    zc = D.read_result(out)
    res["zero_copy_coeffs_equal"] = list(zc.coeffs[:4]) == list(ref.coeffs[:4])
except Exception as e:  # noqa: BLE001
    res["zero_copy_error"] = repr(e)
st, r = ctx.fit_host(pinned.data_ptr(), n, 3, 1)
res["fit_host_GBps"] = timed(lambda: ctx.fit_host(pinned.data_ptr(), n, 3, 1))
print(json.dumps(res, indent=1))
