"""GPU parity on the remaining BASELINE configs (SURVEY §8(c) protocol: per-particle outputs of
a1-a4 on every 64th particle vs the oracle; a5-a7 at full N from the GPU's l):
  C3 forest-like grid, 200 keyframes, per-particle keyframe poses, 4 lattice-shifted modes;
  C5 two near-identical floors, 2 x 20 keyframes, particles spread over both floors;
  C4 1,000,000 particles x 8,192-point scan on one device (capacity; sampled parity)."""
import numpy as np
import pytest

import oracle
import paper_2504_18056_b200 as mcs
import synth
from test_gpu_parity import (L_RTOL, ROT_TOL, T_TOL, check_grad_rows, check_slots, orc_cfg,
                             pose_err)

pytestmark = pytest.mark.gpu


def _subsample_parity(s, step, no_death=True):
    kw = dict(posterior_floor=0.0, loglik_rel_floor=-np.inf) if no_death else {}
    idx = np.arange(0, s.N, step, dtype=np.int32)
    kfs = oracle.Keyframes(s.keyframes, s.D, s.r)
    with mcs.Context(s.N, s.K, s.S, neighbor_count=3, loop_recency_gap=s.gap,
                     voxel_resolution=s.r, **kw) as ctx:
        for (m3, c6), d in zip(s.keyframes, s.D):
            ctx.add_keyframe(m3, c6, d)
        ctx.set_particles(s.pose12, s.kf_pose12)
        ge = ctx.eval(s.scan_mean3, s.scan_cov6)
        g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        st = ctx.get_particles()
    pose, kp = s.pose12[idx].copy(), s.kf_pose12[idx].copy()
    oe = oracle.particles(orc_cfg(s), kfs, s.D_now, pose.copy(), kp.copy(), s.scan_mean3,
                          s.scan_cov6, apply_update=False, slots=True)
    check_slots({k: v[idx] for k, v in ge.items()}, oe, s.S)
    ou = oracle.particles(orc_cfg(s), kfs, s.D_now, pose, kp, s.scan_mean3, s.scan_cov6)
    ok = np.abs(ou["loglik"]) > 0
    assert np.all(np.abs(g["loglik"][idx] - ou["loglik"]) <= L_RTOL * np.abs(ou["loglik"]))
    check_grad_rows(g["grad6"][idx], ou["grad6"], g["hess21"][idx], ou["hess36"])
    np.testing.assert_array_equal(g["flags"][idx], ou["flags"])
    ang, dt = pose_err(st["pose12"][idx], pose)
    assert ang.max() <= ROT_TOL and dt.max() <= T_TOL, (ang.max(), dt.max())
    ak, dk = pose_err(st["kf_pose12"][idx].reshape(-1, 12), kp.reshape(-1, 12))
    assert ak.max() <= ROT_TOL and dk.max() <= T_TOL, (ak.max(), dk.max())
    L, e, w, _, _ = oracle.weights(np.zeros(s.N), g["loglik"])
    np.testing.assert_allclose(g["weight"], w, rtol=1e-12, atol=1e-300)
    return g, ou, ok, st


def test_c3_forest_200_keyframes():
    s = synth.c3()
    g, ou, _, st = _subsample_parity(s, 64)
    assert (ou["flags"] & 1).mean() > 0.2  # a real share of particles closes the loop


@pytest.mark.parametrize("kappa,ok", [(0.0, False), (1.0, True), (20.0, True)])
def test_c3_representative_needs_the_unmatched_penalty(kappa, ok):
    """Behaviour, not parity (R8): with unmatched points skipped (kappa = 0, the literal reading)
    a particle one tree pitch off, whose scan points fall outside the forest, scores higher
    because it has fewer (all non-positive) terms; with kappa > 0 per unmatched (point, slot)
    the representative is the true-mode particle."""
    s = synth.c3()
    with mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r,
                     unmatched_penalty=kappa) as ctx:
        for (m3, c6), d in zip(s.keyframes, s.D):
            ctx.add_keyframe(m3, c6, d)
        ctx.set_particles(s.pose12, s.kf_pose12)
        g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        t = ctx.get_particles()["pose12"][g["representative"]].reshape(3, 4)[:, 3]
    assert (np.linalg.norm(t - s.T_gt[:3, 3]) < 0.5) == ok, np.linalg.norm(t - s.T_gt[:3, 3])


def test_c5_two_floors():
    s = synth.c5()
    g, ou, _, st = _subsample_parity(s, 64)
    assert (ou["flags"] & 2).mean() > 0.5   # loop closure updates (a3/a4 run)


def test_c4_one_million_particles_one_device():
    s = synth.c4()
    _subsample_parity(s, 4096)


def _mixed_slots_c2():
    """C2 with gap 15 (old = id <= 4) and the particles in three groups by index mod 3: as built
    (neighbours {0, 1, 2}: every slot old), moved next to keyframe 5 (neighbours {4, 5, 6}: one
    old and two recent slots, R4's mixed case) and next to keyframe 12 (no old neighbour: no
    loop, G empty, gradient exactly 0).  A particle is moved by T_t <- T_k'^i (T_k1^i)^-1 T_t,
    i.e. it keeps its pose relative to its own estimate of the keyframe it was near."""
    import dataclasses

    s = synth.c2()
    T = s.pose12.reshape(-1, 3, 4).astype(np.float64)
    Kp = s.kf_pose12.reshape(s.N, s.K, 3, 4).astype(np.float64)

    def h(A):
        out = np.zeros(A.shape[:-2] + (4, 4))
        out[..., :3, :] = A
        out[..., 3, 3] = 1
        return out

    moved = h(T)
    for grp, k in ((1, 5), (2, 12)):
        sel = np.arange(s.N) % 3 == grp
        moved[sel] = h(Kp[sel, k]) @ np.linalg.inv(h(Kp[sel, 1])) @ h(T[sel])
    pose12 = np.ascontiguousarray(moved[:, :3, :].reshape(s.N, 12).astype(np.float32))
    return dataclasses.replace(s, gap=15, pose12=pose12)


def test_c2_mixed_old_and_recent_slots():
    """R4 on the GPU (Fig.3): H and b over the old slots only, l over all; rows with an
    exactly zero oracle gradient (no old slot) must be exactly zero on the GPU too."""
    s = _mixed_slots_c2()
    g, ou, _, _ = _subsample_parity(s, 64)
    loop = (ou["flags"] & 1) > 0
    assert 0.2 < loop.mean() < 0.9  # both loop and non-loop particles in the sample
    assert not ou["grad6"][~loop].any() and not g["grad6"][np.arange(0, s.N, 64)][~loop].any()
