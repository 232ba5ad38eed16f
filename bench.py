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
result inside the timed region; ``roofline`` is the dominant kernel's
algorithmic bytes (16 B/point) per launch over its CUDA-event duration;
``cpu_baseline`` is the reference's own CPU path (oracle/_ref, compiled from
the reference sources) timed on this host on a bounded sample.

``--impl reference`` runs only the reference CPU path (rank 0) on the same
metric/config and prints its line with ``"impl": "reference"``.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "points/sec and achieved HBM GB/s (% of roofline) for cubic fit, n=4e9, 1/2/4/8 GPU"
UNIT = "points/s"
SEED = 4
SIGMA = 0.1
BYTES_PER_POINT = 16


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--points", dest="n", type=float, default=4e9, help="total points (default 4e9)")
    p.add_argument("--degree", type=int, default=3)
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-sample", type=float, default=1e8, help="points in the CPU baseline sample")
    p.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo only for emulation tests")
    p.add_argument("--share-gpu", action="store_true", help="test-only: map all ranks onto the visible GPUs")
    return p.parse_args()


def load_peaks():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


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
# clocks during the timed region (NVML poller)
# ----------------------------------------------------------------------------

class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok, self.power = [], 0, False, []
        self.max_mhz = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - NVML missing
            self.err = str(e)
        self._stop = threading.Event()
        self.interval_s = float(os.environ.get("LSQ_CLOCK_SAMPLE_MS", "5")) / 1000.0

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
                self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            except Exception:
                pass
            time.sleep(self.interval_s)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples),
                "power_w_median": statistics.median(self.power) if self.power else None,
                "power_w_max": max(self.power) if self.power else None}


# ----------------------------------------------------------------------------
# CPU legs (the reference's own code, compiled from /root/reference into
# oracle/_ref; the oracle's C port if that build is absent)
# ----------------------------------------------------------------------------

def cpu_reference_timing(n_sample: int, degree: int, steps: int, warmup: int, min_seconds: float = 0.0):
    nproc = os.cpu_count() or 1
    # all host threads for the reference's OpenMP region: torchrun exports
    # OMP_NUM_THREADS=1 to every rank, and libgomp reads it when first loaded
    os.environ["OMP_NUM_THREADS"] = str(nproc)
    import oracle
    oracle.build()
    xy = oracle.synth(n_sample, 0, SEED, 3, SIGMA)  # the first n_sample points of the workload
    kind = "reference" if oracle.have_ref() else "port"
    if kind == "reference":
        ds = oracle.RefDataset(xy)
        run = lambda chunks: ds.fit(degree, chunks)  # noqa: E731  accumulate_parallel+build+solve
    else:
        run = lambda chunks: (0,) + oracle.fit_normal(xy, degree, chunks)[1:]  # noqa: E731
    variants = {}
    # the shipped CLI default (cli.cpp:41-44,62) and the best invocation (8 x nproc chunks)
    for label, chunks in (("chunks=nproc", nproc), ("chunks=8*nproc", 8 * nproc)):
        for _ in range(max(1, warmup)):
            run(chunks)
        times = []
        t_start = time.perf_counter()
        while len(times) < steps or (time.perf_counter() - t_start) < min_seconds:
            t0 = time.perf_counter()
            res = run(chunks)
            times.append(time.perf_counter() - t0)
            if len(times) >= 10000:
                break
        variants[label] = {"median_s": statistics.median(times), "steps": len(times),
                           "pts_per_s": n_sample / statistics.median(times), "status": int(res[0])}
    # single-core sequential accumulate on a smaller slice (bounded)
    n_seq = min(n_sample, 20_000_000)
    if kind == "reference":
        ds_seq = oracle.RefDataset(xy[:n_seq])
        t0 = time.perf_counter()
        ds_seq.accumulate(degree)
        seq_s = time.perf_counter() - t0
    else:
        t0 = time.perf_counter()
        oracle.accumulate(xy[:n_seq], degree)
        seq_s = time.perf_counter() - t0
    variants["sequential(1 core)"] = {"pts_per_s": n_seq / seq_s, "sample_points": n_seq}
    best = max(("chunks=nproc", "chunks=8*nproc"), key=lambda k: variants[k]["pts_per_s"])
    del xy
    threads = oracle.max_threads()  # what the OpenMP runtime actually used
    cpu_model = None
    try:
        with open("/proc/cpuinfo") as f:
            cpu_model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
    except OSError:
        pass
    return {"value": variants[best]["pts_per_s"], "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"first {n_sample:.3g} points of the n=4e9 workload (seed {SEED}), degree {degree}; "
                      f"accumulate_parallel + build_normal_system + solve_gaussian, best of {list(variants)[:2]} "
                      f"with {threads} OpenMP threads, median step",
            "invocation": best, "variants": variants, "ms_per_step": variants[best]["median_s"] * 1e3,
            "cpu_model": cpu_model, "nproc": nproc}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_sample = int(args.cpu_sample)
    cb = cpu_reference_timing(n_sample, args.degree, max(1, args.steps), args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cubic fit (m=3), n=4e9 x~U[-1,1) fp64 AoS, reference CPU path on a bounded sample",
                   "n": int(args.n), "degree": args.degree, "sample_points": n_sample, "parallelism": "cpu-omp"},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "invocation", "variants",
                                            "cpu_model", "nproc")},
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
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    from paper_1512_08017_b200 import _capi, device as D, sharded

    n = int(args.n)
    m = args.degree
    lo, hi = sharded.shard_bounds(n, rank, world)
    n_local = hi - lo
    ctx = _capi.context(local)

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
    with ClockSampler(local) as clk:
        ev[0].record(stream)
        for i in range(K):
            step(kev[i])
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
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
            e2e = run_e2e(args, torch, dist, D, _capi, sharded, ctx, xy, dev, world, n, n_local, m, stream)
        except Exception as exc:  # e.g. the host cannot pin the whole input: still print the line
            e2e = {"value": None, "unit": UNIT, "error": f"{type(exc).__name__}: {exc}"[:300]}
    del xy
    torch.cuda.empty_cache()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = load_peaks()
    alg_bytes = BYTES_PER_POINT * n_local
    achieved = alg_bytes / (kernel_avg_ms * 1e-3) / 1e9
    tpp, tsrc = load_profile_traffic()
    fp64_ops = 5 * m * n_local  # (2m-1) DMUL + 2m DADD + 1 DADD + m DFMA per point
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{'cubic' if m == 3 else f'degree-{m}'} fit, n={n:.3g} points x~U[-1,1) fp64 AoS "
                               f"(BASELINE configs[2])", "n": n, "degree": m, "seed": SEED, "sigma": SIGMA,
                   "parallelism": f"shard{world}" if world > 1 else "single",
                   "l2": f"inputs larger than L2 ({16 * n_local / 1e9:.1f} GB per GPU vs 126 MB), no flush needed",
                   "coefficients": [float(v) for v in res.coeffs[: m + 1]], "status": int(res.status),
                   "grid_ctas": ctx.grid_size()},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": (tpp * n_local) if tpp else None, "peak_source": peak_src,
                     "kernel": "lsq::power_sums_kernel<3>", "kernel_ms": kernel_avg_ms,
                     "alg_bytes_per_launch": alg_bytes, "traffic_source": tsrc,
                     "read_only_stream_ceiling_gbs": 7169.8,
                     "frac_of_read_only_ceiling": achieved / 7169.8,
                     "frac_of_nominal_8000gbs": achieved / 8000.0,
                     "fp64": {"achieved_ops_per_s": fp64_ops / (kernel_avg_ms * 1e-3), "peak_ops_per_s": 1.85e13,
                              "frac": fp64_ops / (kernel_avg_ms * 1e-3) / 1.85e13,
                              "peak_source": "tools/microbench.cu DADD throughput on B200 (64/SM/clk)"}},
        "clocks": clk.summary(),
        "gpu_launches": K * (1 if world == 1 else 2),
    }
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu:
        try:
            cb = cpu_reference_timing(int(args.cpu_sample), m, 3, 1, min_seconds=5.0)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "invocation",
                                                         "variants", "cpu_model", "nproc")}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, torch, dist, D, _capi, sharded, ctx, xy, dev, world, n, n_local, m, stream):
    """Same metric through the public host-buffer API: H2D + fit + D2H per step."""
    host =torch.empty((n_local, 2), dtype=torch.float64, pin_memory=True)
    host.copy_(xy)  # D2H of the resident inputs (untimed setup)
    del xy
    torch.cuda.synchronize()
    steps = max(1, args.e2e_steps)
    if world == 1:
        # lsqfit_cuda_fit_host: H2D into context memory, fused kernel, D2H of the result record
        ptr = host.data_ptr()
        st, r = ctx.fit_host(ptr, n_local, m, _capi.SOLVE)  # warm-up (allocates the device buffer)
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            st, r = ctx.fit_host(ptr, n_local, m, _capi.SOLVE)
            times.append(time.perf_counter() - t0)
        wall = sum(times)
        status = int(r.status)
    else:
        dbuf = torch.empty((n_local, 2), dtype=torch.float64, device=dev)
        part = D.empty_result(dev)
        out = D.empty_result(dev)
        hres = torch.empty(_capi.RESULT_BYTES, dtype=torch.uint8, pin_memory=True)

        def one():
            dbuf.copy_(host, non_blocking=True)
            sharded.gpu_fit_sharded(dbuf, m, part=part, out=out)
            hres.copy_(out, non_blocking=True)
            torch.cuda.synchronize()

        one()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        wall = time.perf_counter() - t0
        tt = torch.tensor([wall], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        wall = float(tt[0])
        status = int(_capi.Result.from_buffer_copy(hres.numpy().tobytes()).status)
        del dbuf
    del host
    return {"value": n * steps / wall, "unit": UNIT, "h2d_bytes_per_step": BYTES_PER_POINT * n,
            "d2h_bytes_per_step": _capi.RESULT_BYTES * world, "steps": steps, "status": status,
            "api": "lsqfit_cuda_fit_host (C ABI, pinned host buffer)" if world == 1 else
                   "H2D + device fit + NCCL all-gather + combine + D2H (per rank)",
            "timing": "host wall clock around synchronous calls, max over ranks"}


if __name__ == "__main__":
    main()
