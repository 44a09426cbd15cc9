"""Point-split sweep of a strong-scaling shard on one GPU: C2 scene, n particles, explicit
mcs_config.point_splits P (0 = auto).  python bench/shard_splits.py 12500 0 4 8 12 16"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2504_18056_b200 as mcs  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1])
s = synth.c2(N=n)
for P in [int(a) for a in sys.argv[2:]]:
    ctx = mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r, point_splits=P)
    for (m3, c6), d in zip(s.keyframes, s.D):
        ctx.add_keyframe(m3, c6, d)
    ctx.set_particles(s.pose12, s.kf_pose12)
    ctx.snapshot()
    ctx.set_profiling(True)
    ph = []
    for k in range(12):
        ctx.restore()
        ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, outputs=("loglik",))
        if k >= 4:
            ph.append(ctx.phase_ms())
    med = {key: float(np.median([p[key] for p in ph])) for key in ph[0]}
    print(json.dumps({"particles": n, "point_splits": P, **{k: round(v, 4) for k, v in med.items()}}))
    ctx.close()
