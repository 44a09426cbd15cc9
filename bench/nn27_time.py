import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np, torch, synth, paper_2504_18056_b200 as mcs
s = synth.c2()
c = mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r, corr_mode=1, nn_radius=s.r)
for (m3, c6), d in zip(s.keyframes, s.D): c.add_keyframe(m3, c6, d)
c.set_particles(s.pose12, s.kf_pose12); c.snapshot(); c.set_profiling(True)
ts = []
for k in range(5):
    c.restore(); c.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, outputs=("loglik",)); ts.append(c.phase_ms()["sweep"])
print("nn27 sweep ms", ts)
