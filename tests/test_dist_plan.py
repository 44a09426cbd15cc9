"""Multi-GPU respawn plan (host logic of DESIGN.md §8), checked on CPU against the oracle's
single-process resampler: the per-rank clone counts and the (src rank -> dst rank) transfer
counts must be exactly those implied by the global donor assignment (R18).  Includes a
world-size-2 gloo run where each rank plans from allgathered totals only."""
import math
import os

import numpy as np
import pytest

import oracle
import paper_2504_18056_b200 as mcs


def _inputs(seed, N):
    g = np.random.default_rng(seed)
    e = np.exp(-g.exponential(g.uniform(0.5, 20), N))
    e[g.integers(0, N)] = 1.0
    dead = (g.random(N) < g.uniform(0.05, 0.95)).astype(np.uint8)
    dead[np.argmax(e)] = 0
    e[dead == 0] = np.maximum(e[dead == 0], 1e-8)
    U = int(g.integers(0, 2**32))
    return e, dead, U


def _shards(seed, N, G):
    g = np.random.default_rng(seed + 1000)
    cuts = np.sort(g.choice(np.arange(1, N), G - 1, replace=False)) if G > 1 else []
    return np.split(np.arange(N), cuts)


def _rank_totals(e, dead, idx):
    q = [0 if dead[i] else math.floor(e[i] * 2**32) for i in idx]
    return sum(q), int(dead[idx].sum())


def _expected(e, dead, U, shards):
    donor = oracle.resample(e, dead, U)
    rank_of = np.zeros(len(e), np.int64)
    for r, idx in enumerate(shards):
        rank_of[idx] = r
    G = len(shards)
    clones = np.zeros(G, np.int64)
    send = np.zeros((G, G), np.int64)
    for i in np.nonzero(donor >= 0)[0]:
        clones[rank_of[donor[i]]] += 1
        send[rank_of[donor[i]], rank_of[i]] += 1
    return clones, send


@pytest.mark.parametrize("seed,N,G", [(s, N, G) for s in range(6) for N, G in
                                      ((7, 1), (50, 2), (333, 3), (1000, 5), (4096, 8))])
def test_plan_matches_global_resampler(seed, N, G):
    e, dead, U = _inputs(seed, N)
    shards = _shards(seed, N, G)
    Qg, Dg = zip(*[_rank_totals(e, dead, idx) for idx in shards])
    plan = mcs.plan_ladder(Qg, Dg, U)
    assert plan["status"] == 0 and plan["D"] == int(dead.sum()) == sum(Dg)
    clones, send = _expected(e, dead, U, shards)
    np.testing.assert_array_equal(plan["clones"], clones)
    np.testing.assert_array_equal(mcs.plan_migration(plan["clones"], Dg), send)
    np.testing.assert_array_equal(plan["d_offset"], np.concatenate([[0], np.cumsum(Dg)[:-1]]))


def test_plan_degenerate_and_bad_inputs():
    assert mcs.plan_ladder([0, 0], [3, 1], 5)["status"] == 7
    with pytest.raises(mcs.MCSError):
        mcs.plan_migration([1, 2], [2, 2])


def _gloo_worker(rank, world, port, seed, N, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        e, dead, U = _inputs(seed, N)
        shards = _shards(seed, N, world)
        Qr, Dr = _rank_totals(e, dead, shards[rank])
        mine = torch.tensor([Qr, Dr], dtype=torch.int64)  # Q < 2^63 here (N * 2^32)
        allv = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allv, mine)
        Qg = [int(v[0]) for v in allv]
        Dg = [int(v[1]) for v in allv]
        plan = mcs.plan_ladder(Qg, Dg, U)
        send = mcs.plan_migration(plan["clones"], Dg)
        clones, send_ref = _expected(e, dead, U, shards)
        ok = (np.array_equal(plan["clones"], clones) and np.array_equal(send, send_ref))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2_plan():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, 3, 5000, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}


def _transport_worker(rank, world, port, q):
    import ctypes as C

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = mcs.TorchDistTransport()
        s = tr.struct
        ok = True
        # allreduce: sum and max of f64, sum of i64, reduced in rank order
        v = np.array([0.1 * (rank + 1), -1.0 * rank, 1e-17], np.float64)
        ok &= s.allreduce(None, rank, v.ctypes.data, 3, 0, 0) == 0
        ref = sum(np.array([0.1 * (r + 1), -1.0 * r, 1e-17]) for r in range(world))
        ok &= np.array_equal(v, ref)
        m = np.array([float(rank), -float(rank)])
        ok &= s.allreduce(None, rank, m.ctypes.data, 2, 0, 1) == 0 and m.tolist() == [1.0, 0.0]
        iv = np.array([rank + 5], np.int64)
        ok &= s.allreduce(None, rank, iv.ctypes.data, 1, 1, 0) == 0 and int(iv[0]) == 11
        # allgather of 5 bytes
        sb = np.full(5, rank + 1, np.uint8)
        rb = np.zeros(5 * world, np.uint8)
        ok &= s.allgather(None, rank, sb.ctypes.data, rb.ctypes.data, 5) == 0
        ok &= rb.tolist() == [1] * 5 + [2] * 5
        # alltoallv with ragged sizes (rank r sends r + p + 1 bytes to p, valued 10r + p)
        send = [np.full(rank + p + 1, 10 * rank + p, np.uint8) for p in range(world)]
        recv = [np.zeros(p + rank + 1, np.uint8) for p in range(world)]
        sp = (C.c_void_p * world)(*[a.ctypes.data for a in send])
        rp = (C.c_void_p * world)(*[a.ctypes.data for a in recv])
        sbs = (C.c_size_t * world)(*[len(a) for a in send])
        rbs = (C.c_size_t * world)(*[len(a) for a in recv])
        ok &= s.alltoallv(None, rank, sp, sbs, rp, rbs) == 0
        ok &= all(np.all(recv[p] == 10 * p + rank) for p in range(world))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_torch_dist_transport_gloo_world_size_2():
    """The mcs_transport callbacks over torch.distributed (gloo), called through their C
    function pointers exactly as libmcs calls them."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_transport_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}
