"""GPU, >= 2 DISTINCT devices (skipped on a 1-GPU box): the multi-GPU paths of
SURVEY §8(e) on real peers, each bit-identical to its single-process local
emulation (per-shard fused kernel + ordered combine on one device):

* one process per GPU over NCCL: sharded.gpu_fit_sharded (fused kernel on the
  rank's shard -> all_gather_into_tensor of the 1016-byte records -> combine +
  solve on every rank), the reference's ascending chunk combine
  (power_sums.cpp:80-87) with ranks as chunks;
* single-process device groups (csrc/api_group.cu) with distinct device ids:
  lsqfit_cuda_group_fit_device (device-resident shards, records peer-copied
  to device 0 over NVLink where the pair has peer access) and
  lsqfit_cuda_group_fit_host (one host dataset split over each GPU's own
  PCIe link).

The NCCL communicator log stays visible (NCCL_DEBUG=INFO in the workers)."""
import os
import socket

import numpy as np
import pytest

from conftest import bitwise_equal

pytestmark = pytest.mark.gpu

N, M, SEED = 40_000_003, 3, 4


def n_gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


needs2 = pytest.mark.skipif("n_gpus() < 2", reason="needs >= 2 distinct GPUs")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def local_emulation(world, m, dev="cuda:0"):
    """Per-shard fused kernel (SUMS) + ordered record combine, on one device."""
    import torch
    from paper_1512_08017_b200 import _capi, device as D, sharded
    parts = D.empty_result(dev, world)
    B = _capi.RESULT_BYTES
    for g in range(world):
        lo, hi = sharded.shard_bounds(N, g, world)
        D.fit(D.synth(hi - lo, lo, SEED, 3, 0.1, device=dev), m, flags=_capi.SUMS, out=parts[g * B:(g + 1) * B])
    r = D.read_result(D.combine(parts, world, m))
    torch.cuda.synchronize()
    return r


def nccl_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NCCL_DEBUG="INFO")
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_1512_08017_b200 import device as D, sharded
        lo, hi = sharded.shard_bounds(N, rank, world)
        xy = D.synth(hi - lo, lo, SEED, 3, 0.1, device=f"cuda:{rank}")
        out = sharded.gpu_fit_sharded(xy, M)
        torch.cuda.synchronize()
        r = D.read_result(out)
        q.put((rank, torch.cuda.current_device(), r.status, r.n, list(r.s[:7]), list(r.t[:4]), list(r.coeffs[:4])))
    finally:
        dist.destroy_process_group()


@needs2
@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_ranks_on_distinct_gpus_equal_local_emulation(world):
    import torch.multiprocessing as mp
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=nccl_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert [r[1] for r in res] == list(range(world))  # each rank on its own device
    ref = local_emulation(world, M)
    for r in res:  # every rank holds the same bits, equal to the emulation
        assert r[2] == 0 and r[3] == N
        assert bitwise_equal(r[4], list(ref.s[:7])) and bitwise_equal(r[5], list(ref.t[:4]))
        assert bitwise_equal(r[6], list(ref.coeffs[:4]))


@needs2
def test_device_group_distinct_devices_fit_device():
    import torch
    from paper_1512_08017_b200 import _capi, device as D, sharded
    G = min(n_gpus(), 8)
    shards = []
    for g in range(G):
        lo, hi = sharded.shard_bounds(N, g, G)
        shards.append(D.synth(hi - lo, lo, SEED, 3, 0.1, device=f"cuda:{g}"))
    for g in range(G):
        torch.cuda.synchronize(g)
    grp = _capi.Group(list(range(G)))
    try:
        st, r = grp.fit_device([s.data_ptr() for s in shards], [s.shape[0] for s in shards], M, _capi.SOLVE)
        st2, r2 = grp.fit_device([s.data_ptr() for s in shards], [s.shape[0] for s in shards], M, _capi.SOLVE)
    finally:
        grp.close()
    assert st == 0 and st2 == 0 and r.n == N
    ref = local_emulation(G, M)
    assert bitwise_equal(list(r.s[:7]), list(ref.s[:7])) and bitwise_equal(list(r.t[:4]), list(ref.t[:4]))
    assert bitwise_equal(list(r.coeffs[:4]), list(ref.coeffs[:4]))
    assert bitwise_equal(list(r.coeffs[:4]), list(r2.coeffs[:4]))
    if torch.cuda.can_device_access_peer(0, 1):
        print("peer access 0<->1 available: records travelled over NVLink")


@needs2
def test_device_group_distinct_devices_fit_host(oracle_mod):
    """One host dataset split over G GPUs (each streams its slice over its
    own link): equal to the same group emulated on device 0, bit for bit."""
    from paper_1512_08017_b200 import _capi
    G = min(n_gpus(), 8)
    xy = oracle_mod.synth(N, 0, SEED, 3, 0.1)
    grp = _capi.Group(list(range(G)))
    emu = _capi.Group([0] * G)
    try:
        st, r = grp.fit_host(xy.ctypes.data, N, M, _capi.SOLVE)
        st2, e = emu.fit_host(xy.ctypes.data, N, M, _capi.SOLVE)
    finally:
        grp.close()
        emu.close()
    assert st == 0 and st2 == 0 and r.n == N
    assert bitwise_equal(list(r.s[:7]), list(e.s[:7])) and bitwise_equal(list(r.coeffs[:4]), list(e.coeffs[:4]))
    s_hi, s_lo, _, t_hi, t_lo, _ = oracle_mod.exact_sums(xy, M)
    st, ex = oracle_mod.solve_from_sums(s_hi + s_lo, t_hi + t_lo, M)
    assert np.max(np.abs(np.array(r.coeffs[:4]) - ex) / np.abs(ex)) <= 1e-10
