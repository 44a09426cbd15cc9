"""C3 (forest, 200 keyframes, 4 modes: a mix of loop and non-loop slots) update time."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_18056_b200 as mcs
import synth
s = synth.c3()
with mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r) as c:
    for (m3, c6), d in zip(s.keyframes, s.D):
        c.add_keyframe(m3, c6, d)
    c.set_particles(s.pose12, s.kf_pose12)
    c.snapshot()
    c.set_profiling(True)
    ph = []
    for k in range(6):
        c.restore()
        c.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, outputs=())
        if k >= 2:
            ph.append(c.phase_ms())
print(json.dumps({k: float(np.median([p[k] for p in ph])) for k in ph[0]}))
