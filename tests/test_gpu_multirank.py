"""Multi-rank path on ONE device: G contexts, one per rank, in G host threads
joined by the in-process transport (host-side collectives only: no kernel ever waits on
another).  Over the same global particle ordering the G-rank result must equal the 1-rank
result bit for bit in every per-particle output except `weight` (S is summed in a rank-order
that differs from the single-device tree), where 1e-12 relative is allowed."""
import threading

import numpy as np
import pytest

import paper_2504_18056_b200 as mcs
import synth

pytestmark = pytest.mark.gpu


def _run_ranks(s, splits, **kw):
    G = len(splits)
    tr = mcs.InprocTransport(G) if G > 1 else None
    results = [None] * G
    errors = []

    def worker(r):
        try:
            idx = splits[r]
            cfg = dict(neighbor_count=3, loop_recency_gap=s.gap, voxel_resolution=s.r,
                       world_size=G, rank=r)
            cfg.update(kw)
            if tr is not None:
                cfg["transport"] = tr
            with mcs.Context(max(len(idx), 1), s.K, s.S, **cfg) as ctx:
                for (m3, c6), d in zip(s.keyframes, s.D):
                    ctx.add_keyframe(m3, c6, d)
                ctx.set_particles(s.pose12[idx], s.kf_pose12[idx])
                out = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, raise_degenerate=False)
                out.update(ctx.get_particles())
                out["p2p"] = ctx.peer_migration_state
                results[r] = out
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append((r, repr(e)))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not errors, errors
    cat = {}
    for k in ("loglik", "grad6", "hess21", "psi6", "weight", "donor", "flags", "pose12",
              "kf_pose12", "L"):
        cat[k] = np.concatenate([res[k] for res in results])
    for k in ("representative", "n_dead", "status", "p2p"):
        vals = {res[k] for res in results}
        assert len(vals) == 1, (k, vals)
        cat[k] = vals.pop()
    return cat


def _check_equal(a, b):
    for k in ("loglik", "grad6", "hess21", "psi6", "donor", "flags", "pose12", "kf_pose12", "L"):
        assert np.array_equal(a[k], b[k]), k
    np.testing.assert_allclose(a["weight"], b["weight"], rtol=1e-12, atol=1e-300)
    assert a["representative"] == b["representative"] and a["n_dead"] == b["n_dead"]


@pytest.mark.parametrize("pm", [1, 0])
@pytest.mark.parametrize("G", [2, 3, 4])
def test_multirank_equals_single_rank_c1(G, pm):
    """pm = 1: clones written straight into the peer context's memory by the draws kernel;
    pm = 0: packed + exchanged through the transport's alltoallv."""
    s = synth.c1()
    N = s.N
    one = _run_ranks(s, [np.arange(N)])
    cuts = np.linspace(0, N, G + 1).astype(int)
    cuts[1:-1] += np.arange(1, G) * 7  # uneven shards
    many = _run_ranks(s, [np.arange(cuts[r], cuts[r + 1]) for r in range(G)],
                      peer_migration=pm)
    assert one["n_dead"] > 0
    assert many["p2p"] == (1 if pm else -1)
    _check_equal(many, one)


@pytest.mark.parametrize("pm", [1, 0])
def test_multirank_migration_heavy(pm):
    """Most particles dead and every survivor on rank 0: clones cross ranks."""
    s = synth.c1()
    N = s.N
    one = _run_ranks(s, [np.arange(N)], posterior_floor=1e-3)
    many = _run_ranks(s, [np.arange(0, 300), np.arange(300, 700), np.arange(700, N)],
                      posterior_floor=1e-3, peer_migration=pm)
    assert many["p2p"] == (1 if pm else -1)
    _check_equal(many, one)
    donor = one["donor"]
    assert (donor >= 0).sum() == one["n_dead"]


def test_exchange_path_with_one_rank_matches_plain():
    """world_size 1 through the in-process transport and through a 1-rank NCCL communicator:
    every exchange step runs and must leave the single-device result unchanged (bitwise)."""
    s = synth.c1()
    N = s.N
    plain = _run_ranks(s, [np.arange(N)])
    tr = mcs.InprocTransport(1)
    with mcs.Context(N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r,
                     transport=tr) as ctx:
        for (m3, c6), d in zip(s.keyframes, s.D):
            ctx.add_keyframe(m3, c6, d)
        ctx.set_particles(s.pose12, s.kf_pose12)
        a = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        a.update(ctx.get_particles())
    for k in ("loglik", "weight", "donor", "flags", "pose12", "kf_pose12", "L"):
        assert np.array_equal(a[k], plain[k]), k
    try:
        nid = mcs.nccl_unique_id()
    except mcs.MCSError:
        pytest.skip("libnccl.so.2 not loadable")
    with mcs.Context(N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r,
                     nccl_unique_id=nid) as ctx:
        for (m3, c6), d in zip(s.keyframes, s.D):
            ctx.add_keyframe(m3, c6, d)
        ctx.set_particles(s.pose12, s.kf_pose12)
        b = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        b.update(ctx.get_particles())
    for k in ("loglik", "weight", "donor", "flags", "pose12", "kf_pose12", "L"):
        assert np.array_equal(b[k], plain[k]), k


def test_nccl_exchange_path_is_graph_captured():
    """With NCCL (here a 1-rank communicator: gpurun gives one GPU) and peer-direct migration
    the exchange steps are device-resident: the library captures the whole update, the
    collectives included, into its CUDA graph, and the caller can capture mcs_update_async into
    its own graph; both replay bitwise equal to kernel-by-kernel updates."""
    import torch
    s = synth.c1()
    try:
        nid = mcs.nccl_unique_id()
    except mcs.MCSError:
        pytest.skip("libnccl.so.2 not loadable")
    runs = {}
    for gr in (0, 1):
        with mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r,
                         nccl_unique_id=mcs.nccl_unique_id(), graph_replay=gr) as ctx:
            for (m3, c6), d in zip(s.keyframes, s.D):
                ctx.add_keyframe(m3, c6, d)
            ctx.set_particles(s.pose12, s.kf_pose12)
            outs = [ctx.update(s.scan_mean3, s.scan_cov6, s.D_now + 0.1 * k,
                               (s.U + 977 * k) & 0xFFFFFFFF) for k in range(3)]
            outs.append(ctx.get_particles())
            assert ctx.peer_migration_state == 1
            assert ctx.graph_captured == bool(gr)
        runs[gr] = outs
    for a, b in zip(runs[0], runs[1]):
        for k in a:
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
    dev = torch.device("cuda", 0)
    ctx = mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r,
                      nccl_unique_id=nid, graph_replay=0)
    for (m3, c6), d in zip(s.keyframes, s.D):
        ctx.add_keyframe(m3, c6, d)
    ctx.set_particles(s.pose12, s.kf_pose12)
    ctx.snapshot()
    d_m = torch.from_numpy(s.scan_mean3).to(dev)
    d_c = torch.from_numpy(s.scan_cov6).to(dev)
    out = {"loglik": torch.zeros(s.N, dtype=torch.float64, device=dev),
           "weight": torch.zeros(s.N, dtype=torch.float64, device=dev),
           "donor": torch.zeros(s.N, dtype=torch.int32, device=dev),
           "representative": torch.zeros(1, dtype=torch.int32, device=dev),
           "n_dead": torch.zeros(1, dtype=torch.int64, device=dev)}
    stream = torch.cuda.Stream(device=dev)
    ctx.set_stream(stream)
    with torch.cuda.stream(stream):
        ctx.update_async(d_m, d_c, s.D_now, s.U, out, stream=stream)
    torch.cuda.synchronize()
    eager = {k: v.clone() for k, v in out.items()}
    eager_state = ctx.get_particles()
    g = torch.cuda.CUDAGraph()
    ctx.restore()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
        ctx.update_async(d_m, d_c, s.D_now, s.U, out, stream=stream)
    for _ in range(2):
        ctx.restore()
        torch.cuda.synchronize()
        for v in out.values():
            v.zero_()
        g.replay()
        torch.cuda.synchronize()
        for k in out:
            assert torch.equal(out[k], eager[k]), k
        st = ctx.get_particles()
        for k in ("pose12", "kf_pose12", "L"):
            np.testing.assert_array_equal(st[k], eager_state[k])
    ctx.close()
