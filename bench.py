#!/usr/bin/env python
"""Benchmark of the normal-equation fit hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

Workload (BASELINE.json configs[2], the metric's config): cubic (m = 3) fit of
n = 4e9 synthetic fp64 (x, y) points, x ~ U[-1, 1), y = cubic + 0.1 z
(counter-based generator, identical bits on host and device; seed 4).
N = 1 holds all 64 GB on one B200; N > 1 shards contiguously (strong scaling:
n fixed), each rank generates its own shard on device.

One step = the whole fit of one batch: the fused power-sums + grid-reduction
(+ solve) kernel; for N > 1 the per-shard kernel, one NCCL all-gather of the
1016-byte partial records, and the combine + solve kernel.

Rank 0 prints ONE JSON line. ``value`` is device-timed (CUDA events, max over
ranks) whole-job points/s with inputs resident in HBM; ``e2e`` is the same
metric through the C ABI with host (pinned) inputs, H2D and the D2H of the
result inside the timed region (median step); ``roofline`` is the dominant
kernel's algorithmic bytes (16 B/point) per launch over its CUDA-event
duration; ``cpu_baseline`` is the reference's own CPU path (oracle/_ref,
compiled from the reference sources) timed on this host over the WHOLE n = 4e9
workload, shard-streamed as BASELINE.md §3 states.

``--impl reference`` runs only the reference CPU path (rank 0) on the same
metric/config and prints its line with ``"impl": "reference"``.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "points/sec and achieved HBM GB/s (% of roofline) for cubic fit, n=4e9, 1/2/4/8 GPU"
UNIT = "points/s"
SEED = 4
SIGMA = 0.1
BYTES_PER_POINT = 16
REF_SHARD = 250_000_000  # host shards of the reference CPU path (<= 2.5e8 points)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--points", dest="n", type=float, default=4e9, help="total points (default 4e9)")
    p.add_argument("--degree", type=int, default=3)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-steps", type=int, default=2, help="timed steps of the CPU baseline leg (ours)")
    p.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo only for emulation tests")
    p.add_argument("--share-gpu", action="store_true", help="test-only: map all ranks onto the visible GPUs")
    return p.parse_args()


def kernel_fp64_ops(m):
    """FP64 operations per point the fused kernel issues for its terms
    (compensation excluded): the reference's rounded terms (m <= 2) cost
    (2m - 1) power multiplies + 2m adds + m moment multiplies + (m + 1) adds
    = 6m; the product terms (m >= 3) (m - 1) power multiplies + one add or
    DFMA per column (3m + 1) = 4m."""
    from paper_1512_08017_b200 import _capi
    if m == 0:
        return 1
    return 4 * m if _capi.sum_terms(m) == _capi.TERMS_PRODUCTS else 6 * m


def config_of(n: int, m: int) -> dict:
    """The workload both arms run (identical dicts: same config)."""
    name = "cubic" if m == 3 else f"degree-{m}"
    return {"workload": f"{name} fit, n={n:.3g} points x~U[-1,1) fp64 AoS (BASELINE configs[2])",
            "n": n, "degree": m, "seed": SEED, "sigma": SIGMA,
            "l2": "inputs larger than L2 (16 B/point x n >> 126 MB), no flush needed"}


def load_peaks():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def load_ceilings() -> dict:
    """Read-only stream ceiling and FP64 pipe peaks measured on a B200 by
    tools/measure_ceilings.py (profiles/measured_ceilings.json); if that file
    is absent, the round-1 probe log profiles/r01_microbench.txt."""
    path = os.path.join(HERE, "profiles", "measured_ceilings.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return {"read_stream_gbs": float(d["read_stream_gbs"]), "dadd_ops_per_s": float(d["dadd_ops_per_s"]),
                "dfma_ops_per_s": float(d["dfma_ops_per_s"]), "source": f"profiles/measured_ceilings.json ({d['how']})"}
    except Exception:
        out = {"source": "profiles/r01_microbench.txt (round-1 probes)"}
        with open(os.path.join(HERE, "profiles", "r01_microbench.txt")) as f:
            for ln in f:
                if not ln.startswith("{"):
                    continue
                r = json.loads(ln)
                if r.get("probe") == "dadd":
                    out["dadd_ops_per_s"] = r["ops_per_s"]
                elif r.get("probe") == "dfma":
                    out["dfma_ops_per_s"] = r["ops_per_s"]
                elif r.get("probe") == "read_stream_ldg128":
                    out["read_stream_gbs"] = r["GB_per_s"]
        return out


def load_profile_traffic():
    """dram bytes per launch per point from the committed ncu --set full capture."""
    path = os.path.join(HERE, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["dram_bytes_per_point"]), d.get("source", path)
    except Exception:
        return None, None


# ----------------------------------------------------------------------------
# clocks during the timed region: a separate sampler PROCESS (no GIL contention
# with the launching thread), NVML clock + throttle reasons every interval,
# timestamped on CLOCK_MONOTONIC; the samples inside [start, stop] are kept.
# ----------------------------------------------------------------------------

_SAMPLER = r"""
import sys, time, json, select
import pynvml as nv
nv.nvmlInit()
ident, interval = sys.argv[1], float(sys.argv[2])
h = nv.nvmlDeviceGetHandleByUUID(ident) if ident.startswith("GPU-") else nv.nvmlDeviceGetHandleByIndex(int(ident))
print(json.dumps({"max": nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)}), flush=True)
rows, k = [], 0
while True:
    t = time.monotonic()
    c = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
    r = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
    p = nv.nvmlDeviceGetPowerUsage(h) / 1000.0 if k % 8 == 0 else None
    rows.append((t, c, r, p))
    k += 1
    if select.select([sys.stdin], [], [], max(0.0, t + interval - time.monotonic()))[0]:
        break
print(json.dumps({"rows": rows}), flush=True)
"""


class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, torch_device):
        import torch
        self.interval_s = float(os.environ.get("LSQ_CLOCK_SAMPLE_MS", "2")) / 1000.0
        self.rows, self.max_mhz, self.err, self.t0, self.t1 = [], None, None, None, None
        try:
            ident = "GPU-" + str(torch.cuda.get_device_properties(torch_device).uuid)
        except Exception:
            ident = str(torch_device.index or 0)
        try:
            self.p = subprocess.Popen([sys.executable, "-c", _SAMPLER, ident, str(self.interval_s)],
                                      stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)
            self.max_mhz = json.loads(self.p.stdout.readline())["max"]
        except Exception as e:  # pragma: no cover - NVML missing
            self.p, self.err = None, str(e)

    def start(self):
        self.t0 = time.monotonic()

    def stop(self):
        self.t1 = time.monotonic()
        if self.p is None:
            return
        try:
            out, _ = self.p.communicate("stop\n", timeout=60)
            self.rows = json.loads(out.strip().splitlines()[-1])["rows"]
        except Exception as e:  # pragma: no cover
            self.err = str(e)
            self.p.kill()

    def summary(self):
        if self.p is None or not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [f"nvml unavailable: {self.err}"]}
        inside = [r for r in self.rows if self.t0 <= r[0] <= self.t1]
        use = inside or self.rows
        mask = 0
        for r in use:
            mask |= r[2]
        gaps = [b[0] - a[0] for a, b in zip(use, use[1:])]
        power = [r[3] for r in use if r[3] is not None]
        return {"sm_mhz": statistics.median(r[1] for r in use), "sm_max_mhz": self.max_mhz,
                "reasons": [v for k, v in self.REASONS.items() if mask & k and k != 0x1],
                "samples": len(inside), "region_s": self.t1 - self.t0,
                "max_gap_ms": max(gaps) * 1e3 if gaps else None,
                "sm_mhz_min": min(r[1] for r in use), "sm_mhz_max": max(r[1] for r in use),
                "power_w_median": statistics.median(power) if power else None,
                "power_w_max": max(power) if power else None,
                "sampler": f"separate process, NVML every {self.interval_s * 1e3:.0f} ms"}


# ----------------------------------------------------------------------------
# The reference's own CPU path (oracle/_ref: compiled from the reference's
# unmodified sources; the oracle's C port only if that build is absent) over
# the WHOLE workload: the n points live on the host as reference Datasets of
# <= 2.5e8 points (built untimed), each step runs accumulate_parallel on every
# shard (timed), adds the shards' sums in ascending order (the additivity of
# test_accumulator.cpp:108-122) and solves once (build_normal_system +
# solve_gaussian) — BASELINE.md §3.
# ----------------------------------------------------------------------------

class ReferenceWorkload:
    def __init__(self, n: int, degree: int):
        nproc = os.cpu_count() or 1
        # all host threads for the reference's OpenMP region: torchrun exports
        # OMP_NUM_THREADS=1 to every rank, and libgomp reads it when first loaded
        os.environ["OMP_NUM_THREADS"] = str(nproc)
        import numpy as np
        import oracle
        oracle.build()
        self.np, self.oracle, self.n, self.m, self.nproc = np, oracle, n, degree, nproc
        self.kind = "reference" if oracle.have_ref() else "port"
        t0 = time.perf_counter()
        self.shards = []
        for lo in range(0, n, REF_SHARD):
            xy = oracle.synth(min(REF_SHARD, n - lo), lo, SEED, 3, SIGMA)
            self.shards.append(oracle.RefDataset(xy) if self.kind == "reference" else xy)
            del xy
        self.setup_s = time.perf_counter() - t0

    def step(self, chunks: int):
        """One fit of the whole workload -> (seconds, status, coefficients)."""
        np, O, m = self.np, self.oracle, self.m
        s, t = np.zeros(2 * m + 1), np.zeros(m + 1)
        t0 = time.perf_counter()
        for sh in self.shards:
            if self.kind == "reference":
                st, ps, pt = sh.accumulate_parallel(m, chunks) if chunks > 1 else sh.accumulate(m)
            else:
                st, ps, pt = O.accumulate_parallel(sh, m, chunks)
            if st != 0:
                return time.perf_counter() - t0, st, None
            s += ps
            t += pt
        st, c = O.ref_solve_from_sums(s, t, m) if self.kind == "reference" else O.solve_from_sums(s, t, m)
        return time.perf_counter() - t0, st, c

    def first_shard_sequential(self):
        """accumulate (one core, the reference's sequential path) on the first
        shard only: reported, not the value (a full pass takes ~20 s)."""
        sh = self.shards[0]
        t0 = time.perf_counter()
        if self.kind == "reference":
            sh.accumulate(self.m)
            k = sh.n
        else:
            self.oracle.accumulate(sh, self.m)
            k = len(sh)
        return k / (time.perf_counter() - t0), k

    def close(self):
        for sh in self.shards:
            if self.kind == "reference":
                sh.close()
        self.shards = []


def cpu_reference_timing(n: int, degree: int, steps: int, warmup: int):
    """Time the reference CPU path on the whole workload: the best invocation
    (chunks = 8 * nproc, which avoids the reference's false sharing) for
    `steps` steps after `warmup`, and the shipped CLI default (chunks = nproc,
    cli.cpp:41-44,62) for one step after one warm-up."""
    W = ReferenceWorkload(n, degree)
    variants = {}
    for label, chunks, k, w in (("chunks=8*nproc", 8 * W.nproc, max(1, steps), max(0, warmup)),
                                ("chunks=nproc", W.nproc, 1, 1)):
        for _ in range(w):
            W.step(chunks)
        times = []
        for _ in range(k):
            dt, st, c = W.step(chunks)
            times.append(dt)
        med = statistics.median(times)
        variants[label] = {"median_s": med, "steps": len(times), "pts_per_s": n / med, "status": int(st),
                           "coefficients": [float(v) for v in c] if c is not None else None}
    rate, k = W.first_shard_sequential()
    variants["sequential(1 core)"] = {"pts_per_s": rate, "sample_points": k,
                                      "note": "accumulate on the first shard only"}
    W.close()
    best = max(("chunks=nproc", "chunks=8*nproc"), key=lambda v: variants[v]["pts_per_s"])
    threads = W.oracle.max_threads()  # what the OpenMP runtime actually used
    cpu_model = None
    try:
        with open("/proc/cpuinfo") as f:
            cpu_model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
    except OSError:
        pass
    return {"value": variants[best]["pts_per_s"], "unit": UNIT, "cores": threads, "kind": W.kind,
            "sample": f"the whole workload: n={n:.3g} points (seed {SEED}) as {len(range(0, n, REF_SHARD))} "
                      f"host shards of <= {REF_SHARD:.3g} (reference Datasets, built untimed in "
                      f"{W.setup_s:.1f} s); per step accumulate_parallel on every shard, ascending shard "
                      f"combine, build_normal_system + solve_gaussian; {threads} OpenMP threads; median step",
            "invocation": best, "variants": variants, "ms_per_step": variants[best]["median_s"] * 1e3,
            "cpu_model": cpu_model, "nproc": W.nproc}


CPU_KEYS = ("value", "unit", "cores", "kind", "sample", "invocation", "variants", "cpu_model", "nproc")


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = int(args.n)
    cb = cpu_reference_timing(n, args.degree, max(1, args.steps), args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": cb["variants"][cb["invocation"]]["steps"], "warmup": args.warmup,
        "ms_per_step": cb["ms_per_step"], "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "parallelism": "cpu-omp",
        "config": config_of(n, args.degree),
        "cpu_baseline": {k: cb[k] for k in CPU_KEYS},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.share_gpu:
        # test-only emulation of N ranks on fewer GPUs: kernels never wait on
        # each other (the exchange is a host-staged gloo all-gather)
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            # keep NCCL's communicator log (transport, NVLS/NVLink rings) on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    from paper_1512_08017_b200 import _capi, device as D, sharded

    n = int(args.n)
    m = args.degree
    lo, hi = sharded.shard_bounds(n, rank, world)
    n_local = hi - lo
    ctx = _capi.context(local)
    clk = ClockSampler(dev)  # the sampler process starts (and imports NVML) before any timing

    # ---- inputs resident in HBM (generated on device, untimed) -------------
    xy = D.synth(n_local, lo, SEED, 3, SIGMA, device=dev)
    part = D.empty_result(dev)
    out = D.empty_result(dev)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream(dev)

    def step(k_ev=None):
        if world == 1:
            if k_ev:
                k_ev[0].record(stream)
            D.fit(xy, m, flags=_capi.SOLVE, out=out)
            if k_ev:
                k_ev[1].record(stream)
        else:
            if k_ev:
                k_ev[0].record(stream)
            D.fit(xy, m, flags=_capi.SUMS, out=part)
            if k_ev:
                k_ev[1].record(stream)
            gathered = sharded.all_gather_records(part)
            D.combine(gathered, world, m, flags=_capi.SOLVE, out=out)

    def barrier():
        if world > 1:
            dist.barrier()

    args.warmup = max(args.warmup, 3)  # timing rule: >= 3 untimed warm-up steps
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    K = args.steps
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    barrier()
    torch.cuda.synchronize()
    clk.start()
    ev[0].record(stream)
    for i in range(K):
        step(kev[i])
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    clk.stop()
    barrier()
    total_ms = ev[0].elapsed_time(ev[K])
    kernel_ms = [a.elapsed_time(b) for a, b in kev]
    res = D.read_result(out)

    t = torch.tensor([total_ms, statistics.mean(kernel_ms)], dtype=torch.float64,
                     device=dev if args.dist_backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kernel_avg_ms = float(t[0]), float(t[1])
    value = n * K / (total_ms * 1e-3)

    # ---- end to end through the C ABI with host (pinned) inputs -------------
    e2e = None
    if not args.no_e2e:
        try:
            e2e = run_e2e(args, torch, dist, D, _capi, sharded, ctx, xy, dev, world, n, n_local, m)
        except Exception as exc:  # e.g. the host cannot pin the whole input: still print the line
            e2e = {"value": None, "unit": UNIT, "error": f"{type(exc).__name__}: {exc}"[:300]}
    del xy
    torch.cuda.empty_cache()
    if hasattr(torch._C, "_host_emptyCache"):
        torch._C._host_emptyCache()  # give the pinned staging back before the CPU leg

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = load_peaks()
    ceil = load_ceilings()
    alg_bytes = BYTES_PER_POINT * n_local
    achieved = alg_bytes / (kernel_avg_ms * 1e-3) / 1e9
    tpp, tsrc = load_profile_traffic()
    fp64_ops = 5 * m * n_local  # (2m-1) DMUL + 2m DADD + 1 DADD + m DFMA per point
    fp64_rate = fp64_ops / (kernel_avg_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (counter-based generator, generated on device, untimed)",
        "parallelism": f"shard{world}" if world > 1 else "single",
        "config": config_of(n, m),
        "result": {"coefficients": [float(v) for v in res.coeffs[: m + 1]], "status": int(res.status),
                   "grid_ctas": ctx.grid_size()},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": (tpp * n_local) if tpp else None, "peak_source": peak_src,
                     "kernel": f"lsq::power_sums_kernel<{m}>", "kernel_ms": kernel_avg_ms,
                     "alg_bytes_per_launch": alg_bytes, "traffic_source": tsrc,
                     "read_only_stream_ceiling_gbs": ceil["read_stream_gbs"],
                     "frac_of_read_only_ceiling": achieved / ceil["read_stream_gbs"],
                     "frac_of_nominal_8000gbs": achieved / 8000.0,
                     "ceilings_source": ceil["source"],
                     "fp64": {"achieved_ops_per_s": fp64_rate, "peak_ops_per_s": ceil["dadd_ops_per_s"],
                              "frac": fp64_rate / ceil["dadd_ops_per_s"],
                              "ops_per_point": 5 * m, "ops_basis": "SURVEY 8(d) algorithmic 5m per point",
                              "kernel_ops_per_point": kernel_fp64_ops(m),
                              "peak_source": "DADD throughput, " + ceil["source"]}},
        "clocks": clk.summary(),
        "gpu_launches": K * (1 if world == 1 else 2),
    }
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu:
        try:
            cb = cpu_reference_timing(n, m, args.cpu_steps, 1)
            line["cpu_baseline"] = {k: cb[k] for k in CPU_KEYS}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": f"{type(e).__name__}: {e}"[:300]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, torch, dist, D, _capi, sharded, ctx, xy, dev, world, n, n_local, m):
    """Same metric through the public host-buffer API: H2D + fit + D2H per
    step, timed per step (host clock around synchronous calls, max over
    ranks); the value is n over the median step."""
    host = torch.empty((n_local, 2), dtype=torch.float64, pin_memory=True)
    host.copy_(xy)  # D2H of the resident inputs (untimed setup)
    torch.cuda.synchronize()
    steps = max(3, args.e2e_steps)
    times = []
    if world == 1:
        # lsqfit_cuda_fit_host: H2D into context memory, fused kernel, D2H of the result record
        ptr = host.data_ptr()
        st, r = ctx.fit_host(ptr, n_local, m, _capi.SOLVE)  # warm-up (allocates the device buffer)
        for _ in range(steps):
            t0 = time.perf_counter()
            st, r = ctx.fit_host(ptr, n_local, m, _capi.SOLVE)
            times.append(time.perf_counter() - t0)
        status = int(r.status)
        api = "lsqfit_cuda_fit_host (C ABI, pinned host buffer)"
    else:
        # each rank: lsqfit_cuda_fit_host on its shard (H2D over its own
        # PCIe link + fused sums, the 1016-byte record back to the host), the
        # record to the device, NCCL all-gather, ordered combine + solve, D2H
        ptr = host.data_ptr()
        part = D.empty_result(dev)
        out = D.empty_result(dev)
        hres = torch.empty(_capi.RESULT_BYTES, dtype=torch.uint8, pin_memory=True)
        hrec = torch.empty(_capi.RESULT_BYTES, dtype=torch.uint8, pin_memory=True)

        def one():
            st_, rec = ctx.fit_host(ptr, n_local, m, _capi.SUMS)
            hrec.copy_(torch.frombuffer(bytearray(bytes(rec)), dtype=torch.uint8))
            part.copy_(hrec, non_blocking=True)
            gathered = sharded.all_gather_records(part)
            D.combine(gathered, world, m, flags=_capi.SOLVE, out=out)
            hres.copy_(out, non_blocking=True)
            torch.cuda.synchronize()

        one()
        for _ in range(steps):
            dist.barrier()
            t0 = time.perf_counter()
            one()
            tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                              device=dev if args.dist_backend == "nccl" else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            times.append(float(tt[0]))
        status = int(_capi.Result.from_buffer_copy(hres.numpy().tobytes()).status)
        api = ("lsqfit_cuda_fit_host per rank (C ABI, pinned host shard, SUMS) + NCCL all-gather of the "
               "records + lsqfit_cuda_combine_device + D2H")
    del host
    med = statistics.median(times)
    return {"value": n / med, "unit": UNIT,
            "h2d_bytes_per_step": BYTES_PER_POINT * n + (_capi.RESULT_BYTES * world if world > 1 else 0),
            "d2h_bytes_per_step": _capi.RESULT_BYTES * world * (2 if world > 1 else 1), "steps": steps, "status": status,
            "median_s": med, "step_s": times, "mean_value": n / statistics.mean(times), "api": api,
            "timing": "host clock around each synchronous step, max over ranks; value = n / median step"}


if __name__ == "__main__":
    main()
