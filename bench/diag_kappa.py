import sys; sys.path.insert(0, '/root/repo')
import numpy as np, synth, paper_2504_18056_b200 as mcs
for name in ("c3", "c5"):
    s = getattr(synth, name)()
    for kappa in (0.0, 1.0, 5.0, 20.0, 100.0):
        with mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r, unmatched_penalty=kappa) as c:
            for (m3, c6), d in zip(s.keyframes, s.D): c.add_keyframe(m3, c6, d)
            c.set_particles(s.pose12, s.kf_pose12)
            ev = c.eval(s.scan_mean3, s.scan_cov6)
            g = c.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
            st = c.get_particles()
        rep = g["representative"]; t = st["pose12"][rep].reshape(3,4)[:,3]
        n = ev["slot_n"].sum(1); l = ev["slot_loglik"].sum(1)
        print(name, kappa, "rep", rep, "mode", rep // (s.N//4), "dist %.3f" % np.linalg.norm(t - s.T_gt[:3,3]), "dz %.2f" % (t[2]-s.T_gt[2,3]),
              "l/n true-mode %.2f" % np.median(l[:1000]/np.maximum(n[:1000],1)), "n true %d other %d" % (np.median(n[:s.N//4]), np.median(n[3*s.N//4:])), flush=True)
