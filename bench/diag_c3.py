"""Diagnostic: C3 pose-parity outliers (psi norms, conditioning, flags)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, synth
import paper_2504_18056_b200 as mcs
s = synth.c3()
idx = np.arange(0, s.N, 64, dtype=np.int32)
kw = dict(posterior_floor=0.0, loglik_rel_floor=-np.inf)
with mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r, **kw) as ctx:
    for (m3, c6), d in zip(s.keyframes, s.D):
        ctx.add_keyframe(m3, c6, d)
    ctx.set_particles(s.pose12, s.kf_pose12)
    g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
    st = ctx.get_particles()
kfs = oracle.Keyframes(s.keyframes, s.D, s.r)
cfg = oracle.make_config(voxel_resolution=s.r, loop_recency_gap=s.gap, **kw)
pose, kp = s.pose12[idx].copy(), s.kf_pose12[idx].copy()
ou = oracle.particles(cfg, kfs, s.D_now, pose, kp, s.scan_mean3, s.scan_cov6, slots=True)
np.savez_compressed("gpurun_out/diag_c3.npz", idx=idx, g_pose=st["pose12"][idx], o_pose=pose,
                    g_psi=g["psi6"][idx], o_psi=ou["psi6"], g_grad=g["grad6"][idx], o_grad=ou["grad6"],
                    g_hess=g["hess21"][idx], o_hess=ou["hess36"], flags=ou["flags"], g_flags=g["flags"][idx],
                    slot_n=ou["slot_n"], o_l=ou["loglik"], g_l=g["loglik"][idx])
print("saved")
