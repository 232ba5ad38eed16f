"""Dev probe: sustained power / SM clock of the fit kernel vs a plain read-only
stream (torch.sum over the same 64 GB) — is the sw_power_cap throttle driven by
HBM traffic or by the FP64 work?"""
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv  # noqa: E402
import torch  # noqa: E402

from paper_1512_08017_b200 import device as D  # noqa: E402


def sample(fn, seconds=4.0):
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    clk, pw, rs = [], [], 0
    stop = threading.Event()

    def poll():
        nonlocal rs
        while not stop.is_set():
            clk.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            pw.append(nv.nvmlDeviceGetPowerUsage(h) / 1000)
            rs |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
            time.sleep(0.01)

    fn()
    torch.cuda.synchronize()
    t = threading.Thread(target=poll)
    t.start()
    t0 = time.time()
    iters = 0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    while time.time() - t0 < seconds:
        for _ in range(10):
            fn()
            iters += 1
        torch.cuda.synchronize()
    ev1.record()
    torch.cuda.synchronize()
    stop.set()
    t.join()
    ms = ev0.elapsed_time(ev1) / iters
    tail = len(clk) // 2  # steady state: second half
    return {"ms_per_iter": ms, "sm_mhz_median_2nd_half": statistics.median(clk[tail:]),
            "power_w_median_2nd_half": statistics.median(pw[tail:]), "power_w_max": max(pw),
            "reasons_mask": hex(rs)}


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 4_000_000_000
    xy = D.synth(n, 0, 4, 3, 0.1)
    out = D.empty_result(xy.device)
    res = {}
    res["fit_m3"] = sample(lambda: D.fit(xy, 3, out=out))
    res["fit_m3"]["GB_per_s"] = 16 * n / (res["fit_m3"]["ms_per_iter"] * 1e-3) / 1e9
    res["fit_m1"] = sample(lambda: D.fit(xy, 1, out=out))
    res["fit_m1"]["GB_per_s"] = 16 * n / (res["fit_m1"]["ms_per_iter"] * 1e-3) / 1e9
    flat = xy.view(-1)
    acc = torch.empty((), dtype=torch.float64, device=xy.device)
    res["torch_sum_read"] = sample(lambda: torch.sum(flat, 0, out=acc))
    res["torch_sum_read"]["GB_per_s"] = 16 * n / (res["torch_sum_read"]["ms_per_iter"] * 1e-3) / 1e9
    time.sleep(3)
    res["fit_m8"] = sample(lambda: D.fit(xy, 8, out=out))
    res["fit_m8"]["GB_per_s"] = 16 * n / (res["fit_m8"]["ms_per_iter"] * 1e-3) / 1e9
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
