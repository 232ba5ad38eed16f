"""Determinism soak: many back-to-back launches of each feed mode (producer
warp m=3, self-feed m=5, self-feed + column split m=8, m=12) on the same data;
every result record must be bit-identical (a pipeline race would show up as
a differing sum). usage: python tools/determinism_soak.py [n] [launches]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1512_08017_b200 import _capi, device as D  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 4_000_000_000
launches = int(sys.argv[2]) if len(sys.argv) > 2 else 300
xy = D.synth(n, 0, 4, 3, 0.1)
out = {"n": n, "launches_per_degree": launches}
for m in (0, 1, 2, 3, 4, 5, 6, 7, 8, 12):  # 0..3 include the dynamic tail
    ref = D.fit(xy, m)
    torch.cuda.synchronize()
    ref_bytes = ref.clone()
    B = _capi.RESULT_BYTES
    # zero-filled like the reference record, so fields past this degree compare equal
    outs = torch.zeros(launches * B, dtype=torch.uint8, device="cuda")
    for i in range(launches):
        D.fit(xy, m, out=outs[i * B:(i + 1) * B])
    torch.cuda.synchronize()
    same = bool((outs.view(launches, B) == ref_bytes.view(1, B)).all().item())
    out[f"m={m}"] = {"all_bit_identical": same, "status": D.read_result(ref).status}
    print(json.dumps({"m": m, "all_bit_identical": same}), flush=True)
print(json.dumps(out))
