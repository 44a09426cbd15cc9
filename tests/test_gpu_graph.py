"""The whole single-GPU update (a1-a7, scan preparation included) is capturable into a CUDA
graph: mcs_update_async issues only stream-ordered work (no host synchronisation, stream-ordered
allocations, CUB calls on the stream).  Replays equal eager updates bitwise."""
import numpy as np
import pytest

import paper_2504_18056_b200 as mcs
import synth

pytestmark = pytest.mark.gpu


def test_update_graph_replay_equals_eager():
    import torch
    s = synth.c1()
    dev = torch.device("cuda", 0)
    ctx = mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r)
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
        ctx.update_async(d_m, d_c, s.D_now, s.U, out, stream=stream)  # eager (warm-up too)
    torch.cuda.synchronize()
    eager = {k: v.clone() for k, v in out.items()}
    eager_state = ctx.get_particles()
    g = torch.cuda.CUDAGraph()
    ctx.restore()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=stream):
        ctx.update_async(d_m, d_c, s.D_now, s.U, out, stream=stream)
    for _ in range(3):
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


def test_library_graph_replay_equals_launch_by_launch():
    """graph_replay = 1 (the library's own captured update body, replayed while the shape holds;
    recaptured when the particle or keyframe count changes) vs 0 (kernel by kernel): several
    consecutive updates with different D_now and U, bitwise equal."""
    s = synth.c1()
    runs = {}
    for gr in (0, 1):
        with mcs.Context(s.N, 4, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r,
                         graph_replay=gr) as ctx:
            for (m3, c6), d in zip(s.keyframes, s.D):
                ctx.add_keyframe(m3, c6, d)
            ctx.set_particles(s.pose12, s.kf_pose12)
            outs = []
            for k in range(3):
                outs.append(ctx.update(s.scan_mean3, s.scan_cov6, s.D_now + 0.1 * k,
                                       (s.U + 977 * k) & 0xFFFFFFFF))
            ctx.set_particles(s.pose12[:700], s.kf_pose12[:700])  # new shape: recapture
            outs.append(ctx.update(s.scan_mean3[:400], s.scan_cov6[:400], s.D_now, s.U))
            m3, c6 = s.keyframes[0]
            ctx.add_keyframe(m3, c6, s.D_now)                     # K changes: recapture
            outs.append(ctx.update(s.scan_mean3, s.scan_cov6, s.D_now + 1.0, s.U ^ 0x5555))
            outs.append(ctx.get_particles())
        runs[gr] = outs
    for a, b in zip(runs[0], runs[1]):
        for k in a:
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
