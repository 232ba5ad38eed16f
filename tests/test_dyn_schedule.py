"""CPU: the power-sum kernel's dynamic-tail schedule (csrc/power_sums.cuh,
dyn_plan + dyn_chunk) partitions the dynamic tiles exactly once for many
(tiles, grid, fraction, chunk) shapes — host-only C++ compiled with nvcc
(no GPU needed)."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)


def test_dynamic_tail_schedule_partitions_tiles(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = tmp_path / "dyn_schedule_check"
    subprocess.run([nvcc, "-std=c++17", "-O2", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-I", os.path.join(REPO, "include"), os.path.join(HERE, "dyn_schedule_check.cu"),
                    "-o", str(exe)], check=True, capture_output=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
