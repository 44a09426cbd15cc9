"""Keyframe-table budget sweep (mcs_config.kf_table_mib) on a config's update phases:
    python bench/table_budget.py c2 8 16 32 64 128"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2504_18056_b200 as mcs  # noqa: E402
import synth  # noqa: E402

s = {"c2": synth.c2, "c3": synth.c3}[sys.argv[1]]()
for mib in [int(a) for a in sys.argv[2:]]:
    ctx = mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r,
                      kf_table_mib=mib)
    for (m3, c6), d in zip(s.keyframes, s.D):
        ctx.add_keyframe(m3, c6, d)
    ctx.set_particles(s.pose12, s.kf_pose12)
    ctx.snapshot()
    ctx.set_profiling(True)
    ph = []
    for k in range(10):
        ctx.restore()
        ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, outputs=("loglik",))
        if k >= 3:
            ph.append(ctx.phase_ms())
    med = {key: round(float(np.median([p[key] for p in ph])), 4) for key in ph[0]}
    print(json.dumps({"config": sys.argv[1], "kf_table_mib": mib, **med}))
    ctx.close()
