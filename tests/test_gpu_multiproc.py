"""Two processes on one device, one rank each, joined by torch.distributed (gloo) through
mcs.TorchDistTransport: the multi-process exchange path, including the peer-direct migration
over CUDA IPC mappings of the other process's state (no kernel waits on another process; the
ranks meet only at host barriers).  The result must equal the single-rank run bitwise."""
import os

import numpy as np
import pytest

import paper_2504_18056_b200 as mcs
import synth

pytestmark = pytest.mark.gpu
SPLIT = 420  # uneven shards


def _worker(rank, port, pm, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        s = synth.c1()
        idx = np.arange(0, SPLIT) if rank == 0 else np.arange(SPLIT, s.N)
        with mcs.Context(len(idx), s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r,
                         posterior_floor=1e-3, world_size=2, rank=rank, device=0,
                         transport=mcs.TorchDistTransport(), peer_migration=pm) as ctx:
            for (m3, c6), d in zip(s.keyframes, s.D):
                ctx.add_keyframe(m3, c6, d)
            ctx.set_particles(s.pose12[idx], s.kf_pose12[idx])
            out = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
            out.update(ctx.get_particles())
            out["p2p"] = ctx.peer_migration_state
            dist.barrier()  # no rank unmaps its buffers while the other may still write
        q.put((rank, out))
    except Exception as e:  # pragma: no cover - reported by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("pm", [1, 0])
def test_two_processes_equal_single_rank(pm):
    import torch.multiprocessing as mp
    s = synth.c1()
    with mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r,
                     posterior_floor=1e-3) as ctx:
        for (m3, c6), d in zip(s.keyframes, s.D):
            ctx.add_keyframe(m3, c6, d)
        ctx.set_particles(s.pose12, s.kf_pose12)
        one = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        one.update(ctx.get_particles())
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = 31500 + os.getpid() % 1000 + 7 * pm
    procs = [ctxm.Process(target=_worker, args=(r, port, pm, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(60)
    assert all(isinstance(res[r], dict) for r in range(2)), res
    assert res[0]["p2p"] == res[1]["p2p"] == (1 if pm else -1)
    for k in ("loglik", "grad6", "psi6", "donor", "flags", "pose12", "kf_pose12", "L"):
        got = np.concatenate([res[0][k], res[1][k]])
        assert np.array_equal(got, one[k]), k
    np.testing.assert_allclose(np.concatenate([res[0]["weight"], res[1]["weight"]]),
                               one["weight"], rtol=1e-12, atol=1e-300)
    assert res[0]["representative"] == one["representative"]
    assert (one["donor"] >= 0).sum() == one["n_dead"] > 0
