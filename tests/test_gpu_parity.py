"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded
synthetic scenes, at the north-star tolerances:
  l to 1e-4 relative, gradient to 1e-3 relative (vector norm), H to 1e-3 (Frobenius),
  poses to 1e-5 rad / 1e-5 m after one step, sum w = 1 +- 1e-12,
  resampled indices bit-exact given the same fp64 e and uniform.
"""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
import paper_2504_18056_b200 as mcs
import synth

pytestmark = pytest.mark.gpu

L_RTOL, G_RTOL, H_RTOL, ROT_TOL, T_TOL = 1e-4, 1e-3, 1e-3, 1e-5, 1e-5


def make_ctx(s, N=None, **kw):
    N = s.N if N is None else N
    cfg = dict(neighbor_count=3, loop_recency_gap=s.gap, voxel_resolution=s.r)
    cfg.update(kw)
    ctx = mcs.Context(N, max(s.K, 1), max(s.S, 1), **cfg)
    for (m3, c6), d in zip(s.keyframes, s.D):
        ctx.add_keyframe(m3, c6, d)
    ctx.set_particles(s.pose12[:N], s.kf_pose12[:N])
    return ctx


def orc_cfg(s, **kw):
    c = dict(voxel_resolution=s.r, loop_recency_gap=s.gap)
    c.update(kw)
    return oracle.make_config(**c)


def rel_err(a, b, axis=None):
    num = np.linalg.norm(np.asarray(a, float) - b, axis=axis)
    den = np.linalg.norm(np.asarray(b, float), axis=axis)
    return num / np.maximum(den, 1e-30)


def pose_err(P, Q):
    P = np.asarray(P, float).reshape(-1, 3, 4)
    Q = np.asarray(Q, float).reshape(-1, 3, 4)
    Rrel = np.einsum("nji,njk->nik", Q[:, :, :3], P[:, :, :3])
    ang = np.linalg.norm(Rotation.from_matrix(Rrel).as_rotvec(), axis=1)
    return ang, np.linalg.norm(P[:, :, 3] - Q[:, :, 3], axis=1)


def check_grad_rows(g_grad, o_grad, g_h21, o_h36):
    """Gradient rows at G_RTOL (vector norm) and H at H_RTOL (Frobenius) where the oracle's row
    is nonzero; where it is exactly zero (G empty: no old slot, R4) the GPU row must be exactly
    zero as well, so a leak of non-G slots into g or H cannot hide behind a mask."""
    nz = np.linalg.norm(o_grad, axis=1) > 0
    assert np.all(rel_err(g_grad[nz], o_grad[nz], axis=1) <= G_RTOL)
    assert not np.asarray(g_grad)[~nz].any(), "nonzero GPU gradient where the oracle's is 0"
    Hg = mcs.unpack_h21(g_h21).reshape(-1, 36).astype(float)
    Ho = np.asarray(o_h36).reshape(-1, 36)
    hz = np.linalg.norm(Ho, axis=1) > 0
    assert np.all(rel_err(Hg[hz], Ho[hz], axis=1) <= H_RTOL)
    assert not Hg[~hz].any(), "nonzero GPU H where the oracle's is 0"


def check_slots(g, o, S):
    """g: mcs_eval outputs; o: oracle slot outputs for the same particles."""
    np.testing.assert_array_equal(g["slot_kf"], o["slot_kf"])
    np.testing.assert_array_equal(g["slot_n"], o["slot_n"])
    lg, lo = g["slot_loglik"], o["slot_l"]
    assert np.all(np.abs(lg - lo) <= L_RTOL * np.abs(lo))
    Hg = mcs.unpack_h21(g["slot_H21"]).astype(float)
    Ho = o["slot_H36"]
    active = o["slot_n"] > 0
    eH = rel_err(Hg.reshape(Hg.shape[:2] + (36,)), Ho.reshape(Ho.shape[:2] + (36,)), axis=-1)
    assert np.all(eH[active] <= H_RTOL), eH[active].max()
    eb = rel_err(g["slot_b6"], o["slot_b6"], axis=-1)
    assert np.all(eb[active] <= G_RTOL), eb[active].max()


# ---------------------------------------------------------------- C1 (full N)
@pytest.fixture(scope="module")
def c1():
    return synth.c1()


def test_eval_c1_full_parity(c1):
    s = c1
    with make_ctx(s) as ctx:
        g = ctx.eval(s.scan_mean3, s.scan_cov6)
    o = oracle.particles(orc_cfg(s), oracle.Keyframes(s.keyframes, s.D, s.r), s.D_now,
                         s.pose12.copy(), s.kf_pose12.copy(), s.scan_mean3, s.scan_cov6,
                         apply_update=False, slots=True)
    check_slots(g, o, s.S)
    np.testing.assert_array_equal(g["loop"], o["flags"] & 1)
    assert (g["slot_n"][:, 0] > 0).mean() > 0.99


def _no_death(s):
    return dict(posterior_floor=0.0, loglik_rel_floor=-np.inf)


def test_update_c1_parity_without_respawn(c1):
    """Every per-particle output of one update, with the dead set empty (floors off), so the
    poses can be compared particle by particle."""
    s = c1
    with make_ctx(s, **_no_death(s)) as ctx:
        g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        st = ctx.get_particles()
    pose, kp, L = s.pose12.copy(), s.kf_pose12.copy(), np.zeros(s.N)
    o = oracle.update(orc_cfg(s, **_no_death(s)), oracle.Keyframes(s.keyframes, s.D, s.r),
                      s.D_now, pose, kp, L, s.scan_mean3, s.scan_cov6, s.U)
    assert g["n_dead"] == o["n_dead"] == 0
    assert np.all(np.abs(g["loglik"] - o["loglik"]) <= L_RTOL * np.abs(o["loglik"]))
    assert np.all(rel_err(g["grad6"], o["grad6"], axis=1) <= G_RTOL)
    Hg = mcs.unpack_h21(g["hess21"]).reshape(-1, 36)
    assert np.all(rel_err(Hg, o["hess36"].reshape(-1, 36), axis=1) <= H_RTOL)
    np.testing.assert_array_equal(g["flags"], o["flags"])
    ang, dt = pose_err(st["pose12"], pose)
    assert ang.max() <= ROT_TOL and dt.max() <= T_TOL, (ang.max(), dt.max())
    np.testing.assert_array_equal(st["kf_pose12"], kp)  # K = 1: t_o's ratio is 0 -> untouched
    np.testing.assert_allclose(st["L"], L, rtol=L_RTOL)
    assert abs(g["weight"].sum() - 1) < 1e-12
    # weights on a common L: the oracle's Eq.11 normalisation of the GPU's L
    _, _, w_ref, _, _ = oracle.weights(st["L"])
    np.testing.assert_allclose(g["weight"], w_ref, rtol=1e-12, atol=1e-300)
    assert g["representative"] == oracle.representative(w_ref)


def test_update_c1_respawn_from_gpu_loglik(c1):
    """Default floors: the oracle recomputes weights, dead set and donors from the
    GPU's l and the same U; donors, dead count and representative must match exactly."""
    s = c1
    with make_ctx(s) as ctx:
        g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        st = ctx.get_particles()
    L, e, w, _, _ = oracle.weights(np.zeros(s.N), g["loglik"])
    dead, nd = oracle.dead(g["loglik"], w)
    donor = oracle.resample(e, dead, s.U)
    assert g["n_dead"] == nd and nd > 0
    np.testing.assert_array_equal(g["donor"], donor)
    np.testing.assert_array_equal((g["flags"] & 8) > 0, dead > 0)
    for i in np.nonzero(donor >= 0)[0]:
        assert np.array_equal(st["pose12"][i], st["pose12"][donor[i]])
        assert np.array_equal(st["kf_pose12"][i], st["kf_pose12"][donor[i]])
        assert st["L"][i] == st["L"][donor[i]]
    L2 = L.copy()
    L2[donor >= 0] = L[donor[donor >= 0]]
    _, _, w2, _, _ = oracle.weights(L2)
    np.testing.assert_allclose(g["weight"], w2, rtol=1e-12, atol=1e-300)
    assert abs(g["weight"].sum() - 1) < 1e-12
    assert g["representative"] == oracle.representative(w2)


def test_update_is_bitwise_deterministic(c1):
    s = c1
    outs = []
    for _ in range(2):
        with make_ctx(s) as ctx:
            g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
            g.update(ctx.get_particles())
            outs.append(g)
    for k in ("loglik", "grad6", "hess21", "psi6", "weight", "donor", "flags", "pose12",
              "kf_pose12", "L"):
        assert np.array_equal(outs[0][k], outs[1][k]), k


def test_update_async_matches_sync(c1):
    import torch
    s = c1
    with make_ctx(s) as ctx:
        g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
    dev = torch.device("cuda")
    out = {"loglik": torch.zeros(s.N, dtype=torch.float64, device=dev),
           "weight": torch.zeros(s.N, dtype=torch.float64, device=dev),
           "donor": torch.zeros(s.N, dtype=torch.int32, device=dev),
           "representative": torch.zeros(1, dtype=torch.int32, device=dev),
           "n_dead": torch.zeros(1, dtype=torch.int64, device=dev)}
    with make_ctx(s) as ctx:
        stream = torch.cuda.Stream()
        ctx.update_async(torch.from_numpy(s.scan_mean3).to(dev), torch.from_numpy(s.scan_cov6).to(dev),
                         s.D_now, s.U, out, stream=stream)
        stream.synchronize()
    assert np.array_equal(out["loglik"].cpu().numpy(), g["loglik"])
    assert np.array_equal(out["weight"].cpu().numpy(), g["weight"])
    assert np.array_equal(out["donor"].cpu().numpy(), g["donor"])
    assert int(out["representative"][0]) == g["representative"]
    assert int(out["n_dead"][0]) == g["n_dead"]


# ---------------------------------------------------------------- resampler bit-exactness
def test_resample_bit_exact_random():
    g = np.random.default_rng(21)
    with mcs.Context(200_000, 1, 1) as ctx:
        for trial in range(40):
            N = int(g.choice([1, 2, 7, 255, 256, 257, 1000, 4097, 65_537, 200_000]))
            e = np.exp(-g.exponential(g.uniform(0.1, 30), N))
            e[g.integers(0, N)] = 1.0
            dead = (g.random(N) < g.uniform(0, 0.999)).astype(np.uint8)
            dead[np.argmax(e)] = 0
            # the whole domain [0, 1]: zero rungs (e < 2^-32), exact zeros, tiny and unit e
            k = g.integers(0, N, max(1, N // 10))
            e[k] = g.choice([0.0, 2.0**-33, 1e-12, 2.0**-32, 1e-8, 1.0], len(k))
            U = int(g.integers(0, 2**32))
            np.testing.assert_array_equal(ctx.resample(e, dead, U), oracle.resample(e, dead, U))


def test_resample_rejects_values_outside_the_domain():
    """mcs_resample's domain is 0 <= e <= 1 (e = exp(L - max L)): anything else is refused
    before any work, so the bit-exact contract holds wherever the call succeeds."""
    with mcs.Context(16, 1, 1) as ctx:
        dead = np.zeros(4, np.uint8)
        dead[3] = 1
        for bad in (1.5, -1e-300, np.nan, np.inf):
            e = np.array([1.0, 0.5, bad, 0.25])
            with pytest.raises(mcs.MCSError) as ei:
                ctx.resample(e, dead, 7)
            assert ei.value.status == 1
        e = np.array([1.0, 0.0, 2.0**-40, 0.5])  # zero rungs are inside the domain
        np.testing.assert_array_equal(ctx.resample(e, dead, 7), oracle.resample(e, dead, 7))


def test_resample_exact_boundaries():
    with mcs.Context(16, 1, 1) as ctx:
        for N, dead_idx, U in ((3, [2], 2**31), (5, [1, 3], 0), (6, [0, 5], 2**31), (4, [3], 0),
                               (4, [3], 2**32 - 1)):
            e = np.ones(N)
            dead = np.zeros(N, np.uint8)
            dead[dead_idx] = 1
            np.testing.assert_array_equal(ctx.resample(e, dead, U), oracle.resample(e, dead, U))
        # the hand case of tests/golden (R18)
        e = np.array([1.0, np.exp(-40.0), np.exp(-10.0)])
        dead = np.array([0, 1, 0], np.uint8)
        assert list(ctx.resample(e, dead, 4294772313)) == [-1, 0, -1]
        assert list(ctx.resample(e, dead, 4294772314)) == [-1, 2, -1]
        with pytest.raises(mcs.MCSError):
            ctx.resample(np.ones(3), np.ones(3, np.uint8), 5)


# ---------------------------------------------------------------- C2 (headline config)
@pytest.fixture(scope="module")
def c2():
    return synth.c2()


def test_c2_subsample_parity(c2):
    """Full C2 (100k particles x 4096 points vs 20 keyframes) in the bench launch
    configuration; per-particle outputs of a1-a4 on every 64th particle vs the oracle."""
    s = c2
    idx = np.arange(0, s.N, 64, dtype=np.int32)
    kfs = oracle.Keyframes(s.keyframes, s.D, s.r)
    with make_ctx(s, **_no_death(s)) as ctx:
        ge = ctx.eval(s.scan_mean3, s.scan_cov6)
        g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        st = ctx.get_particles()
    pose, kp = s.pose12.copy(), s.kf_pose12.copy()
    oe = oracle.particles(orc_cfg(s), kfs, s.D_now, pose, kp, s.scan_mean3, s.scan_cov6,
                          idx=idx, apply_update=False, slots=True)
    check_slots({k: v[idx] for k, v in ge.items()}, oe, s.S)
    ou = oracle.particles(orc_cfg(s), kfs, s.D_now, pose, kp, s.scan_mean3, s.scan_cov6, idx=idx)
    assert np.all(ou["flags"] & 1)  # C2: every particle takes the loop path
    assert np.all(np.abs(g["loglik"][idx] - ou["loglik"]) <= L_RTOL * np.abs(ou["loglik"]))
    assert np.all(rel_err(g["grad6"][idx], ou["grad6"], axis=1) <= G_RTOL)
    np.testing.assert_array_equal(g["flags"][idx], ou["flags"])
    ang, dt = pose_err(st["pose12"][idx], pose[idx])
    assert ang.max() <= ROT_TOL and dt.max() <= T_TOL, (ang.max(), dt.max())
    ak, dk = pose_err(st["kf_pose12"][idx].reshape(-1, 12), kp[idx].reshape(-1, 12))
    assert ak.max() <= ROT_TOL and dk.max() <= T_TOL, (ak.max(), dk.max())
    # a5-a7 at full N from the GPU's l
    L, e, w, _, _ = oracle.weights(np.zeros(s.N), g["loglik"])
    np.testing.assert_allclose(g["weight"], w, rtol=1e-12, atol=1e-300)


def test_c2_respawn_full_n(c2):
    s = c2
    with make_ctx(s) as ctx:
        g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
    L, e, w, _, _ = oracle.weights(np.zeros(s.N), g["loglik"])
    dead, nd = oracle.dead(g["loglik"], w)
    assert g["n_dead"] == nd
    np.testing.assert_array_equal(g["donor"], oracle.resample(e, dead, s.U))


# ---------------------------------------------------------------- edge cases
def test_fewer_keyframes_than_neighbours_and_ragged_scan(c1):
    """K = 2 < 3 slots (min(3, K) used), S = 300 (ragged vs the 256-point stage), N = 333."""
    s = c1
    m3, c6 = s.keyframes[0]
    import dataclasses
    kf_pose = np.concatenate([s.kf_pose12[:333], s.kf_pose12[:333]], axis=1)
    kf_pose[:, 1, 3] += 0.25
    s2 = dataclasses.replace(s, keyframes=[(m3, c6), (m3, c6)], D=np.array([0.0, 1.0]),
                             pose12=np.ascontiguousarray(s.pose12[:333]),
                             kf_pose12=np.ascontiguousarray(kf_pose),
                             scan_mean3=np.ascontiguousarray(s.scan_mean3[:300]),
                             scan_cov6=np.ascontiguousarray(s.scan_cov6[:300]))
    with make_ctx(s2) as ctx:
        g = ctx.eval(s2.scan_mean3, s2.scan_cov6)
    o = oracle.particles(orc_cfg(s2), oracle.Keyframes(s2.keyframes, s2.D, s2.r), 2.0,
                         s2.pose12.copy(), s2.kf_pose12.copy(), s2.scan_mean3, s2.scan_cov6,
                         apply_update=False, slots=True)
    assert np.all(g["slot_kf"][:, 2] == -1)
    check_slots(g, o, 300)


def test_no_match_is_singular_and_single_particle(c1):
    s = c1
    far = synth.to12(synth.pose(t=(5000.0, 0, 0)))[None]
    with mcs.Context(1, 1, s.S, loop_recency_gap=0, voxel_resolution=s.r) as ctx:
        ctx.add_keyframe(*s.keyframes[0], 0.0)
        ctx.set_particles(far, s.kf_pose12[:1])
        g = ctx.update(s.scan_mean3, s.scan_cov6, 1.0, 0)
        assert g["loglik"][0] == 0.0 and g["flags"][0] & 4 and not g["flags"][0] & 2
        assert g["weight"][0] == 1.0 and g["representative"] == 0 and g["n_dead"] == 0


def test_errors_before_state_change(c1):
    s = c1
    with mcs.Context(10, 2, 16, voxel_resolution=s.r) as ctx:
        with pytest.raises(mcs.MCSError) as ei:
            ctx.scan_nonplanar()
        assert ei.value.status == 6  # no scan prepared yet
        with pytest.raises(mcs.MCSError) as ei:
            ctx.update(s.scan_mean3[:16], s.scan_cov6[:16], 1.0, 0)
        assert ei.value.status == 6  # no keyframe
        bad = s.keyframes[0][1][:16].copy()
        bad[3] = [1, 2, 0, 1, 0, 1]   # not positive definite
        with pytest.raises(mcs.MCSError) as ei:
            ctx.add_keyframe(s.keyframes[0][0][:16], bad, 0.0)
        assert ei.value.status == 1 and ctx.sizes == (0, 0)
        ctx.add_keyframe(*s.keyframes[0], 0.0)
        ctx.set_particles(s.pose12[:10], s.kf_pose12[:10])
        with pytest.raises(mcs.MCSError) as ei:
            ctx.update(s.scan_mean3[:17], s.scan_cov6[:17], 1.0, 0)
        assert ei.value.status == 5
        nanscan = s.scan_mean3[:16].copy()
        nanscan[0, 0] = np.nan
        before = ctx.get_particles()
        with pytest.raises(mcs.MCSError) as ei:
            ctx.update(nanscan, s.scan_cov6[:16], 1.0, 0)
        assert ei.value.status == 1
        after = ctx.get_particles()
        assert np.array_equal(before["pose12"], after["pose12"])


def test_path_length_below_newest_keyframe_is_rejected(c1):
    """R14: D is a cumulative path length, so D_now below the newest keyframe's D_k is an
    argument error, reported before any state change."""
    s = c1
    with make_ctx(s) as ctx:
        before = ctx.get_particles()
        with pytest.raises(mcs.MCSError) as ei:
            ctx.update(s.scan_mean3, s.scan_cov6, float(s.D[-1]) - 0.5, s.U)
        assert ei.value.status == 1
        after = ctx.get_particles()
        for k in ("pose12", "kf_pose12", "L"):
            assert np.array_equal(before[k], after[k]), k


def test_all_dead_is_degenerate(c1):
    s = c1
    with make_ctx(s, posterior_floor=2.0) as ctx:
        g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, raise_degenerate=False)
        assert g["status"] == 7 and g["n_dead"] == s.N and np.all(g["donor"] == -1)


def test_c2_degenerate_update_keeps_and_propagates_every_state(c2):
    """S:381 with loop closures: a posterior floor above 1 kills every particle, so a6 skips
    the respawn and every particle keeps its own updated state — including the keyframe poses
    the survivor-only a4 had skipped (propagated after all once the ladder finds no survivor).
    Poses and keyframe poses on every 64th particle vs the oracle's a1-a4."""
    s = c2
    idx = np.arange(0, s.N, 64, dtype=np.int32)
    with make_ctx(s, posterior_floor=2.0) as ctx:
        g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, raise_degenerate=False)
        st = ctx.get_particles()
    assert g["status"] == 7 and g["n_dead"] == s.N and np.all(g["donor"] == -1)
    pose, kp = s.pose12.copy(), s.kf_pose12.copy()
    oracle.particles(orc_cfg(s), oracle.Keyframes(s.keyframes, s.D, s.r), s.D_now, pose, kp,
                     s.scan_mean3, s.scan_cov6, idx=idx)
    assert np.any(kp[idx] != s.kf_pose12[idx])
    ang, dt = pose_err(st["pose12"][idx], pose[idx])
    assert ang.max() <= ROT_TOL and dt.max() <= T_TOL, (ang.max(), dt.max())
    ak, dk = pose_err(st["kf_pose12"][idx].reshape(-1, 12), kp[idx].reshape(-1, 12))
    assert ak.max() <= ROT_TOL and dk.max() <= T_TOL, (ak.max(), dk.max())


def test_c2_survival_variant_respawn_full_n():
    """The C2 survival variant (bench --config c2_survival: particles 1 mm / 0.1 mrad around the
    truth, ~30 % survive P:190's floors): tens of thousands of donors and clones instead of the
    headline's one survivor.  Donors bit-exact against the oracle's resampler fed the GPU's l
    (full N), every clone a copy of its donor's pose, keyframe poses and L, weights on the
    oracle's normalisation of the new L."""
    s = synth.c2(sig_t=1e-3, sig_r=1e-4, drift_t=1e-4, drift_r=1e-5)
    with make_ctx(s) as ctx:
        g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        st = ctx.get_particles()
    L, e, w, _, _ = oracle.weights(np.zeros(s.N), g["loglik"])
    dead, nd = oracle.dead(g["loglik"], w)
    assert g["n_dead"] == nd and 0.2 * s.N < nd < 0.9 * s.N, nd
    donor = oracle.resample(e, dead, s.U)
    np.testing.assert_array_equal(g["donor"], donor)
    assert len(np.unique(donor[donor >= 0])) > 1000  # many distinct donors
    idx = np.nonzero(donor >= 0)[0]
    np.testing.assert_array_equal(st["pose12"][idx], st["pose12"][donor[idx]])
    # a4 runs for the survivors only (a dead particle's keyframe poses are its donor's): the
    # clones carry their donors' propagated keyframe poses, and the survivors' match the
    # oracle's a1-a4 on a subsample
    np.testing.assert_array_equal(st["kf_pose12"][idx], st["kf_pose12"][donor[idx]])
    surv = np.nonzero(donor < 0)[0][::37].astype(np.int32)
    pose, kp = s.pose12.copy(), s.kf_pose12.copy()
    oracle.particles(orc_cfg(s), oracle.Keyframes(s.keyframes, s.D, s.r), s.D_now, pose, kp,
                     s.scan_mean3, s.scan_cov6, idx=surv)
    assert np.any(kp[surv] != s.kf_pose12[surv])  # the oracle propagated them
    ak, dk = pose_err(st["kf_pose12"][surv].reshape(-1, 12), kp[surv].reshape(-1, 12))
    assert ak.max() <= ROT_TOL and dk.max() <= T_TOL, (ak.max(), dk.max())
    np.testing.assert_array_equal(st["kf_pose12"][idx], st["kf_pose12"][donor[idx]])
    np.testing.assert_array_equal(st["L"][idx], st["L"][donor[idx]])
    L2 = L.copy()
    L2[idx] = L[donor[idx]]
    _, _, w2, _, _ = oracle.weights(L2)
    np.testing.assert_allclose(g["weight"], w2, rtol=1e-12, atol=1e-300)
    assert g["representative"] == oracle.representative(w2)
