"""NN27 (R33) update timing on C2: `python bench/nn27_time.py [reps]` (phase events, sweep ms)."""
import sys

sys.path.insert(0, __file__.rsplit("/bench/", 1)[0])
import paper_2504_18056_b200 as mcs  # noqa: E402
import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
s = synth.c2()
c = mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r,
                corr_mode=mcs.CORR_NN27, nn_radius=s.r)
for (m3, c6), d in zip(s.keyframes, s.D):
    c.add_keyframe(m3, c6, d)
c.set_particles(s.pose12, s.kf_pose12)
c.snapshot()
c.set_profiling(True)
ts = []
for k in range(reps):
    c.restore()
    c.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, outputs=("loglik",))
    ts.append(c.phase_ms()["sweep"])
print("nn27 sweep ms", ts)
