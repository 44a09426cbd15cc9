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
