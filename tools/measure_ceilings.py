"""Measure the roofline denominators bench.py and tools/sweep.py divide by,
on the GPU box, and write them to profiles/measured_ceilings.json:

  read_stream_gbs  best read-only HBM stream over two probes:
                   tools/microbench.cu (grid-stride LDG.128, 8 CTAs/SM) and
                   tools/stream_balance.cu (the hot kernel's own feed: a
                   persistent TMA bulk-copy ring, static / dynamic tile deals)
  dadd_ops_per_s   FP64 add throughput (tools/microbench.cu, 8 indep. chains)
  dfma_ops_per_s   FP64 FMA throughput
  nvml_query_ms    latency of one NVML clock + throttle-reason query (sizes
                   bench.py's clock sampler)

    python tools/measure_ceilings.py [out.json]   # builds the probes if needed
"""
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def build(name):
    exe = os.path.join(ROOT, "tools", name)
    src = exe + ".cu"
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.run([NVCC, "-O3", *ARCH, "-o", exe, src], check=True)
    return exe


def run_json_lines(exe):
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600, check=True)
    return [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]


def nvml_latency():
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(0)
        ts = []
        for _ in range(200):
            t0 = time.perf_counter()
            nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            ts.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(ts), max(ts)
    except Exception as e:  # pragma: no cover
        return None, str(e)


def main():
    mb = run_json_lines(build("microbench"))
    sb = run_json_lines(build("stream_balance"))
    by = {r["probe"]: r for r in mb if "probe" in r}
    best_sb = max(sb, key=lambda r: r["GB_per_s"])
    reads = {"ldg128_grid_stride": by["read_stream_ldg128"]["GB_per_s"],
             f"tma_ring ({best_sb['mode']})": best_sb["GB_per_s"]}
    med, worst = nvml_latency()
    import torch
    out = {
        "read_stream_gbs": max(reads.values()),
        "read_stream_probes_gbs": reads,
        "dadd_ops_per_s": by["dadd"]["ops_per_s"],
        "dfma_ops_per_s": by["dfma"]["ops_per_s"],
        "fp64_per_sm_per_clk_at_max": {"dadd": by["dadd"]["per_sm_per_clk_at_max"],
                                       "dfma": by["dfma"]["per_sm_per_clk_at_max"]},
        "nvml_query_ms": {"median": med, "max": worst},
        "device": torch.cuda.get_device_name(0),
        "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
        "how": "tools/measure_ceilings.py: tools/microbench.cu (DADD/DFMA chains, LDG.128 grid-stride read of 32 GiB) "
               "and tools/stream_balance.cu (TMA bulk-copy ring read of 32 GiB, static/dynamic deals); best of passes",
        "raw": {"microbench": mb, "stream_balance": sb},
    }
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "measured_ceilings.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("read_stream_gbs", "read_stream_probes_gbs", "dadd_ops_per_s",
                                          "dfma_ops_per_s", "nvml_query_ms")}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
