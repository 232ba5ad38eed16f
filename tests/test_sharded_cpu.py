"""CPU, world_size 2 over gloo: the multi-GPU host logic (shard bounds, the
single all-gather of lsqfit_result records in rank order, combine) with the
oracle standing in for the device kernels."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N, M, SEED = 100_003, 3, 17


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def record_from_exact(xy, m):
    """An lsqfit_result record (same layout the kernel writes) from oracle dd sums."""
    import oracle
    from paper_1512_08017_b200 import _capi
    r = _capi.Result()
    s_hi, s_lo, _, t_hi, t_lo, _ = oracle.exact_sums(xy, m)
    for v in range(2 * m):
        r.part_hi[v], r.part_lo[v] = s_hi[v + 1], s_lo[v + 1]
    for j in range(m + 1):
        r.part_hi[2 * m + j], r.part_lo[2 * m + j] = t_hi[j], t_lo[j]
    r.n, r.degree = len(xy), m
    return torch.frombuffer(bytearray(bytes(r)), dtype=torch.uint8).clone()


def dd_add(h, l, bh, bl):
    s = h + bh
    bb = s - h
    e = (h - (s - bb)) + (bh - bb)
    e += l + bl
    hh = s + e
    return hh, e - (hh - s)


def combine_records(gathered, world):
    from paper_1512_08017_b200 import _capi
    recs = [_capi.Result.from_buffer_copy(gathered[i * _capi.RESULT_BYTES:(i + 1) * _capi.RESULT_BYTES].numpy().tobytes())
            for i in range(world)]
    out = _capi.Result()
    nv = 3 * M + 1
    for v in range(nv):
        h = l = 0.0
        for r in recs:  # ascending rank order
            h, l = dd_add(h, l, r.part_hi[v], r.part_lo[v])
        out.part_hi[v], out.part_lo[v] = h, l
    out.n = sum(r.n for r in recs)
    return out


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1512_08017_b200 import sharded
        lo, hi = sharded.shard_bounds(N, rank, world)
        xy = oracle.synth(hi - lo, lo, SEED, 3, 0.1)  # each rank generates only its shard
        out = sharded.fit_sharded(lambda a, b: record_from_exact(xy, M), combine_records, N)
        q.put((rank, lo, hi, out.n, [out.part_hi[v] for v in range(3 * M + 1)],
               [out.part_lo[v] for v in range(3 * M + 1)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_sharded_fit_matches_whole(world):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # shards tile [0, N) contiguously in rank order
    assert res[0][1] == 0 and res[-1][2] == N
    assert all(res[i][2] == res[i + 1][1] for i in range(world - 1))
    # every rank combined the same records in the same order: identical bits
    assert all(r[4] == res[0][4] and r[5] == res[0][5] for r in res)
    assert res[0][3] == N
    whole = oracle.synth(N, 0, SEED, 3, 0.1)
    s_hi, s_lo, s_abs, t_hi, t_lo, t_abs = oracle.exact_sums(whole, M)
    ex = np.concatenate([s_hi[1:] + s_lo[1:], t_hi + t_lo])
    ab = np.concatenate([s_abs[1:], t_abs])
    got = np.array(res[0][4]) + np.array(res[0][5])
    assert (np.abs(got - ex) <= 1e-30 * ab + np.spacing(np.abs(ex))).all()


def test_shard_bounds_formula():
    from paper_1512_08017_b200 import sharded
    for n in (0, 1, 7, 4_000_000_000):
        for world in (1, 2, 3, 8):
            spans = [sharded.shard_bounds(n, g, world) for g in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
