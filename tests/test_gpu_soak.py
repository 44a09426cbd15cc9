"""Soak: hundreds of consecutive updates on one context with keyframe insertions, particle-set
changes (graph recaptures) and predictions, then several contexts created and destroyed: no
error, no device-memory growth across contexts."""
import numpy as np
import pytest

import paper_2504_18056_b200 as mcs
import synth

pytestmark = pytest.mark.gpu


def _free_bytes():
    import torch
    torch.cuda.synchronize()
    return torch.cuda.mem_get_info()[0]


def test_soak_updates_and_context_churn():
    s = synth.c1()
    g = np.random.default_rng(0)
    m3, c6 = s.keyframes[0]
    before = None
    for round_ in range(3):
        with mcs.Context(s.N, 8, s.S, loop_recency_gap=2, voxel_resolution=s.r) as ctx:
            ctx.add_keyframe(m3, c6, 0.0)
            ctx.set_particles(s.pose12, s.kf_pose12)
            K = 1
            for k in range(150):
                if k % 50 == 49 and K < 8:
                    ctx.add_keyframe(m3, c6, float(k))
                    K += 1
                if k % 60 == 59:
                    n = int(g.integers(200, s.N + 1))
                    ctx.set_particles(s.pose12[:n], np.repeat(s.kf_pose12[:n], K, axis=1))
                if k % 7 == 0:
                    ctx.predict(synth.to12(np.eye(4)), np.eye(6) * 1e-6, 3, k)
                out = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now + k, int(g.integers(2**32)),
                                 outputs=("weight",), raise_degenerate=False)
                assert abs(out["weight"].sum() - 1.0) < 1e-9 or out["status"] == 7
        free = _free_bytes()
        if before is None:
            before = free
        else:  # contexts 2 and 3 leave the device exactly as context 1 did (pools included)
            assert abs(free - before) < 64 * 2**20, (before, free)
