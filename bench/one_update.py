"""Runs C2 updates (eager, library graph off) for ncu captures of single kernels:
    ncu --set full -k regex:sweep_kernel --launch-skip 1 --launch-count 1 python bench/one_update.py 2
"""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2504_18056_b200 as mcs, synth
s = synth.c2()
with mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r, graph_replay=0) as ctx:
    for (m3, c6), d in zip(s.keyframes, s.D):
        ctx.add_keyframe(m3, c6, d)
    ctx.set_particles(s.pose12, s.kf_pose12)
    ctx.snapshot()
    for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
        ctx.restore()
        ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, outputs=())
print("done")
