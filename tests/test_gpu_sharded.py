"""GPU: the multi-GPU path end to end with 2 ranks sharing one GPU (gloo
exchange, the only emulation allowed on a 1-GPU box: the ranks' kernels never
wait on each other). The distributed result must equal, bit for bit, the
single-process emulation (fit each shard, combine records in rank order), and
every rank must hold the same bits."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import bitwise_equal

pytestmark = pytest.mark.gpu

N, M, SEED = 20_000_011, 3, 4


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1512_08017_b200 import device as D, sharded
        lo, hi = sharded.shard_bounds(N, rank, world)
        xy = D.synth(hi - lo, lo, SEED, 3, 0.1, device="cuda:0")
        out = sharded.gpu_fit_sharded(xy, M)
        torch.cuda.synchronize()
        r = D.read_result(out)
        q.put((rank, r.status, r.n, list(r.s[:7]), list(r.t[:4]), list(r.coeffs[:4])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_equals_local_emulation(world):
    import torch
    from paper_1512_08017_b200 import _capi, device as D, sharded
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in res:
        assert r[1] == 0 and r[2] == N
        assert bitwise_equal(r[3], res[0][3]) and bitwise_equal(r[5], res[0][5])
    # local emulation: per-shard fit (SUMS) + ordered combine
    parts = D.empty_result("cuda:0", world)
    B = _capi.RESULT_BYTES
    for g in range(world):
        lo, hi = sharded.shard_bounds(N, g, world)
        D.fit(D.synth(hi - lo, lo, SEED, 3, 0.1), M, flags=_capi.SUMS, out=parts[g * B:(g + 1) * B])
    comb = D.read_result(D.combine(parts, world, M))
    torch.cuda.synchronize()
    assert bitwise_equal(res[0][3], list(comb.s[:7])) and bitwise_equal(res[0][4], list(comb.t[:4]))
    assert bitwise_equal(res[0][5], list(comb.coeffs[:4]))
    # and close to the unsharded single launch
    whole = D.read_result(D.fit(D.synth(N, 0, SEED, 3, 0.1), M))
    rel = max(abs(a - b) / abs(b) for a, b in zip(res[0][5], whole.coeffs[:4]))
    assert rel <= 1e-12
