"""bench.py keeps the driver's contract: one JSON line with the required keys,
for the reference arm (CPU-only, runs here) and for our arm at N = 1 and, with
two ranks sharing one GPU over gloo (the emulation that keeps kernels
independent), at N = 2 under torchrun."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def run(args, timeout=900, env=None):
    p = subprocess.run(args, cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                       env={**os.environ, **(env or {})})
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    import oracle
    oracle.build()
    # torchrun exports OMP_NUM_THREADS=1 to every rank: the arm must still use every host core
    d = run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1",
             "--points", "6e6"], env={"OMP_NUM_THREADS": "1"})
    assert d["cpu_baseline"]["cores"] == (os.cpu_count() or 1)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # the whole workload, not a prefix: the same config dict our arm prints
    import bench
    assert d["config"] == json.loads(json.dumps(bench.config_of(6_000_000, 3)))
    assert "sample_points" not in d["config"]
    v = d["cpu_baseline"]["variants"]
    assert v["chunks=8*nproc"]["steps"] == 2 and v["chunks=nproc"]["steps"] == 1
    assert all(v[k]["status"] == 0 and len(v[k]["coefficients"]) == 4 for k in ("chunks=8*nproc", "chunks=nproc"))


@pytest.mark.gpu
def test_our_arm_line_single_gpu():
    d = run([sys.executable, "bench.py", "--points", "2e7", "--steps", "3", "--warmup", "3"])
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["result"]["status"] == 0
    import bench
    assert d["config"] == json.loads(json.dumps(bench.config_of(20_000_000, 3)))
    assert d["clocks"]["sm_mhz"] is not None and d["e2e"]["steps"] >= 3
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["achieved"] > 0 and d["gpu_launches"] == 3
    assert d["e2e"]["h2d_bytes_per_step"] == 16 * 20_000_000 and d["e2e"]["status"] == 0
    assert d["cpu_baseline"]["value"] > 0 and "clocks" in d


@pytest.mark.gpu
def test_our_arm_two_ranks_shared_gpu():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    d = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
             "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
             "--points", "2e7", "--steps", "3", "--warmup", "3", "--share-gpu", "--dist-backend", "gloo"])
    assert d["n_gpus"] == 2 and d["result"]["status"] == 0 and d["parallelism"] == "shard2"
    assert d["e2e"]["status"] == 0 and d["gpu_launches"] == 6


def test_reference_arm_under_torchrun_two_ranks():
    """The driver launches --impl reference like our arm (torchrun for N > 1):
    rank 0 alone runs the CPU path and prints the one line; rank 1 exits 0."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    d = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
             "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
             "--gpus", "2", "--points", "3e6", "--steps", "2", "--warmup", "1"])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["cores"] == (os.cpu_count() or 1)
