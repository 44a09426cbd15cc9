"""Pins for the CPU oracle: closed forms, worked examples, invariants and brute force.

Each test fixes a part of the oracle against something other than itself (the
paper's definitions, a library routine, exact rational arithmetic, brute
force), chosen so that a dropped term, a wrong sign or index, or a transposed
operand fails at least one of them.  CPU only.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy.linalg import expm
from scipy.spatial.transform import Rotation

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_cases.json")))


def hat(xi):
    """4x4 twist matrix of xi = (rho, phi) (independent of the oracle)."""
    rho, phi = np.asarray(xi[:3], float), np.asarray(xi[3:], float)
    M = np.zeros((4, 4))
    M[:3, :3] = [[0, -phi[2], phi[1]], [phi[2], 0, -phi[0]], [-phi[1], phi[0], 0]]
    M[:3, 3] = rho
    return M


def T44(T12):
    T = np.eye(4)
    T[:3, :4] = np.asarray(T12, float).reshape(3, 4)
    return T


# --------------------------------------------------------------------- SE(3)
def test_exp_identity_and_quarter_turn():
    assert np.array_equal(oracle.se3_exp(np.zeros(6)), np.eye(4)[:3])
    T = oracle.se3_exp([0, 0, 0, 0, 0, np.pi / 2])
    np.testing.assert_allclose(T[:3, :3], [[0, -1, 0], [1, 0, 0], [0, 0, 1]], atol=1e-15)
    np.testing.assert_allclose(T[:, 3], 0, atol=1e-15)


def test_exp_matches_matrix_exponential():
    g = np.random.default_rng(1)
    for scale in (1e-7, 1e-5, 1e-3, 0.3, 1.0, 2.5):
        for _ in range(20):
            xi = g.normal(size=6)
            xi[3:] *= scale / np.linalg.norm(xi[3:])
            np.testing.assert_allclose(oracle.se3_exp(xi), expm(hat(xi))[:3], atol=2e-13)


def test_log_exp_round_trip():
    g = np.random.default_rng(2)
    worst = 0.0
    for _ in range(1000):
        xi = g.normal(size=6)
        xi[3:] *= g.uniform(0, 3.0) / np.linalg.norm(xi[3:])
        worst = max(worst, np.abs(oracle.se3_log(oracle.se3_exp(xi)) - xi).max())
    assert worst < 1e-9


# --------------------------------------------------------------------- voxel map
def test_cell_floor_not_truncation_and_range():
    assert list(oracle.cell_of([0.1, 0.1, 0.1], 1.0)) == [0, 0, 0]
    assert list(oracle.cell_of([-0.1, 0.0, 0.0], 1.0)) == [-1, 0, 0]
    assert list(oracle.cell_of([-1048576.0, 1048575.5, -0.5], 1.0)) == [-1048576, 1048575, -1]
    assert oracle.cell_of([1048576.0, 0, 0], 1.0) is None
    assert oracle.cell_of([-1048577.0, 0, 0], 1.0) is None
    assert oracle.cell_of([np.nan, 0, 0], 1.0) is None


def test_map_aggregates_mean_of_means():
    m3 = np.array([[0.1, 0.1, 0.1], [0.5, 0.3, 0.9], [-0.1, 0.0, 0.0]], np.float32)
    c6 = np.array([[1, 0, 0, 1, 0, 1], [3, 0, 0, 3, 0, 3], [2, 0, 0, 2, 0, 2]], np.float32)
    m = oracle.Map(m3, c6, 1.0)
    assert len(m) == 2
    cnt, mean, cov = m.lookup([0, 0, 0])
    assert cnt == 2
    np.testing.assert_allclose(mean, (m3[0].astype(float) + m3[1]) / 2, rtol=0, atol=0)
    np.testing.assert_allclose(cov, [2, 0, 0, 2, 0, 2])
    assert m.lookup([-1, 0, 0])[0] == 1
    assert m.lookup([1, 0, 0])[0] == 0


def test_cell_correspondence_equals_brute_force_binning():
    """the lookup equals naive fp32 floor-binning of ALL points."""
    g = np.random.default_rng(3)
    pts = g.uniform(-6, 6, (3000, 3)).astype(np.float32)
    cov = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (3000, 1))
    cov[:, 0] = g.uniform(0.5, 2, 3000)
    r = 0.5
    m = oracle.Map(pts, cov, r)
    cells = np.floor(pts * np.float32(1 / r)).astype(np.int64)
    q = g.uniform(-7, 7, (10000, 3)).astype(np.float32)
    qc = np.floor(q * np.float32(1 / r)).astype(np.int64)
    for k in range(len(q)):
        members = np.nonzero((cells == qc[k]).all(axis=1))[0]
        cnt, mean, cv = m.lookup(qc[k])
        assert cnt == len(members)
        if cnt:
            np.testing.assert_allclose(mean, pts[members].astype(float).mean(0), rtol=1e-15,
                                       atol=1e-15)
            np.testing.assert_allclose(cv, cov[members].astype(float).mean(0), rtol=1e-15)


# --------------------------------------------------------------------- relative pose
def test_relpose_is_inverse_times_current():
    g = np.random.default_rng(4)
    for _ in range(50):
        Tk = synth.pose(g.normal(size=3), g.uniform(-40, 40, 3))
        Tt = synth.pose(g.normal(size=3), g.uniform(-40, 40, 3))
        Tk32, Tt32 = synth.to12(Tk), synth.to12(Tt)
        r32, r64 = oracle.relpose(Tk32, Tt32)
        ref = np.linalg.inv(T44(Tk32)) @ T44(Tt32)  # fp64 (T_k)^-1 T_t of the fp32 inputs
        # rotation part: R_k^T R_t (exact inverse for the orthonormal part of fp32 R_k)
        Rk, Rt = T44(Tk32)[:3, :3], T44(Tt32)[:3, :3]
        np.testing.assert_allclose(r64[:, :3], Rk.T @ Rt, atol=1e-15)
        np.testing.assert_allclose(r64[:, 3], Rk.T @ (T44(Tt32)[:3, 3] - T44(Tk32)[:3, 3]),
                                   atol=1e-12)
        np.testing.assert_allclose(r64, ref[:3], atol=1e-5)  # fp32 R is orthonormal to ~1e-7
        np.testing.assert_allclose(r32, r64, atol=2e-5)


# --------------------------------------------------------------------- likelihood
def _hand():
    h = GOLD["gicp_hand_case"]
    m = oracle.Map(np.array([h["mu_prime"]], np.float32), np.array([h["cov6_prime"]], np.float32),
                   h["r"])
    rel = np.eye(4)[:3].copy()
    rel[:, 3] = h["rel_translation"]
    return h, m, rel


def test_gicp_hand_case():
    h, m, rel = _hand()
    res = oracle.pair_linearize(m, np.array([h["mu"]]), np.array([h["cov6"]]), rel, rel)
    assert res.n == 1 and res.l == h["loglik"]
    np.testing.assert_array_equal(-2 * res.b, h["grad6"])
    np.testing.assert_array_equal(res.H, np.diag(h["H_diag"]))


def test_gicp_hand_case_one_damped_step():
    """Eq.5 + Eq.7 via the full per-particle path (K = 1, gap 0 => loop)."""
    h, m, rel = _hand()
    cfg = oracle.make_config(voxel_resolution=h["r"], loop_recency_gap=0)
    kfs = oracle.Keyframes([(np.array([h["mu_prime"]]), np.array([h["cov6_prime"]]))], [0.0],
                           h["r"])
    pose = synth.to12(T44(rel.reshape(12)))[None].copy()
    kp = synth.to12(np.eye(4))[None, None].copy()
    out = oracle.particles(cfg, kfs, 1.0, pose, kp, np.array([h["mu"]]), np.array([h["cov6"]]))
    assert out["flags"][0] & 2  # updated
    np.testing.assert_allclose(pose[0, 3], h["residual_after_one_damped_step_m"], rtol=1e-6)
    np.testing.assert_allclose(out["psi6"][0], [-1 / (1 + 5e-7), 0, 0, 0, 0, 0], rtol=1e-15)


def _self_scene(seed=0, r=0.25):
    """A box-room cloud downsampled at r: one point per cell, so at the keyframe pose every
    scan point is its own correspondence (Q7/R7)."""
    world = synth.box_room(seed)
    T = synth.pose((0, 0, 0.3), (6.0, 4.5, 1.4))
    m3, c6 = synth.sensor_cloud(world, T, r, None, synth.rng(seed, f"self/{r}"), 720, 160)
    return m3, c6, r


def test_self_match_is_exactly_zero():
    """A scan matched against itself at its keyframe pose: e = 0, l = 0, b = 0 exactly."""
    m3, c6, r = _self_scene()
    m = oracle.Map(m3, c6, r)
    # identity, and a signed permutation with a representable translation
    P = np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1]], float)
    for R, t in ((np.eye(3), np.zeros(3)), (P, np.array([2.0, -3.5, 0.25]))):
        Tt = np.eye(4)
        Tt[:3, :3], Tt[:3, 3] = R, t
        r32, r64 = oracle.relpose(synth.to12(Tt), synth.to12(Tt))
        res = oracle.pair_linearize(m, m3, c6, r32, r64)
        assert res.n == len(m3)
        assert res.l == 0.0 and np.all(res.b == 0.0)


def test_self_match_general_pose_small():
    m3, c6, r = _self_scene()
    m = oracle.Map(m3, c6, r)
    Tt = synth.pose((0.3, -0.2, 1.1), (12.25, -3.3, 0.7))
    r32, r64 = oracle.relpose(synth.to12(Tt), synth.to12(Tt))
    res = oracle.pair_linearize(m, m3, c6, r32, r64)
    assert res.n >= len(m3) - 5
    assert abs(res.l) < 1e-8 * len(m3)


def test_additivity_identical_neighbours_and_slot_sum():
    """Eq.2: the particle log-likelihood is the sum over neighbour keyframes."""
    s = synth.c1()
    m3, c6 = s.keyframes[0]
    cfg = oracle.make_config(voxel_resolution=s.r, loop_recency_gap=0, neighbor_count=3)
    g = np.random.default_rng(5)
    kf_poses = [np.eye(4), np.eye(4), synth.pose((0, 0, 0.05), (0.2, 0.1, 0))]
    kfs = oracle.Keyframes([(m3, c6)] * 3, [0.0, 1.0, 2.0], s.r)
    Tt = synth.pose(g.normal(0, 0.02, 3), g.normal(0, 0.1, 3))
    pose = synth.to12(Tt)[None].copy()
    kp = synth.to12(np.stack(kf_poses))[None].copy()
    out = oracle.particles(cfg, kfs, 3.0, pose, kp, s.scan_mean3, s.scan_cov6,
                           apply_update=False, slots=True)
    singles = []
    for k in range(3):
        r32, r64 = oracle.relpose(kp[0, k], pose[0])
        singles.append(oracle.pair_linearize(kfs.maps[k], s.scan_mean3, s.scan_cov6, r32, r64).l)
    assert singles[0] == singles[1] and singles[0] != 0
    np.testing.assert_allclose(out["loglik"][0], sum(singles), rtol=1e-14)
    assert sorted(out["slot_l"][0]) == sorted(singles)


def test_invariance_under_common_rigid_transform():
    s = synth.c1()
    m = oracle.Map(*s.keyframes[0], s.r)
    Tt = T44(s.pose12[3])
    Tk = T44(s.kf_pose12[3, 0])
    base = oracle.pair_linearize(m, s.scan_mean3, s.scan_cov6, *oracle.relpose(synth.to12(Tk),
                                                                               synth.to12(Tt)))
    G = synth.pose((0.4, -0.3, 0.9), (5.0, -7.0, 1.5))
    moved = oracle.pair_linearize(m, s.scan_mean3, s.scan_cov6,
                                  *oracle.relpose(synth.to12(G @ Tk), synth.to12(G @ Tt)))
    # fp32 rounding of the moved poses may flip a few correspondences near cell faces
    assert abs(moved.n - base.n) <= 3
    np.testing.assert_allclose(moved.l, base.l, rtol=2e-2)


# --------------------------------------------------------------------- gradient and H
def _linearised(seed=6):
    s = synth.c1()
    m = oracle.Map(*s.keyframes[0], s.r)
    g = np.random.default_rng(seed)
    Tk = T44(s.kf_pose12[0, 0])
    Tt = T44(synth.to12(s.T_gt @ synth.pose(g.normal(0, 0.01, 3), g.normal(0, 0.05, 3))))
    r32, r64 = oracle.relpose(synth.to12(Tk), synth.to12(Tt))
    res = oracle.pair_linearize(m, s.scan_mean3, s.scan_cov6, r32, r64)
    om = oracle.pair_omegas(m, s.scan_cov6, r64, res.corr)
    return s, m, r64, res, om


def test_gradient_matches_central_differences():
    """g = -2b = dl/d(delta) with Omega and correspondences frozen (R3), right perturbation."""
    s, m, r64, res, om = _linearised()
    base = T44(r64.reshape(12))
    h = 1e-6
    fd = np.zeros(6)
    for k in range(6):
        d = np.zeros(6)
        d[k] = h
        lp = oracle.pair_loglik_frozen(m, s.scan_mean3, (base @ expm(hat(d)))[:3], res.corr, om)
        lm = oracle.pair_loglik_frozen(m, s.scan_mean3, (base @ expm(hat(-d)))[:3], res.corr, om)
        fd[k] = (lp - lm) / (2 * h)
    assert res.n > 100
    np.testing.assert_allclose(oracle.pair_loglik_frozen(m, s.scan_mean3, r64, res.corr, om),
                               res.l, rtol=1e-12)
    assert np.linalg.norm(-2 * res.b - fd) <= 1e-6 * np.linalg.norm(fd)


def test_H_is_half_hessian_at_zero_residual():
    """At e = 0 the exact Hessian of -l (Omega frozen) is 2 J^T Omega J = 2H (Eq.6)."""
    m3, c6, r = _self_scene()
    m = oracle.Map(m3, c6, r)
    T = np.eye(4)
    r32, r64 = oracle.relpose(synth.to12(T), synth.to12(T))
    res = oracle.pair_linearize(m, m3, c6, r32, r64)
    om = oracle.pair_omegas(m, c6, r64, res.corr)
    h = 1e-4
    f = lambda d: -oracle.pair_loglik_frozen(m, m3, expm(hat(d))[:3], res.corr, om)
    Hfd = np.zeros((6, 6))
    for a in range(6):
        for b in range(6):
            ea, eb = np.eye(6)[a] * h, np.eye(6)[b] * h
            Hfd[a, b] = (f(ea + eb) - f(ea - eb) - f(-ea + eb) + f(-ea - eb)) / (4 * h * h)
    np.testing.assert_allclose(2 * res.H, Hfd, rtol=1e-5, atol=1e-4 * np.abs(Hfd).max())


def test_H_symmetric_psd():
    _, _, _, res, _ = _linearised(7)
    np.testing.assert_allclose(res.H, res.H.T, rtol=1e-13, atol=1e-9)
    assert np.linalg.eigvalsh(res.H).min() > -1e-9 * np.abs(res.H).max()


# --------------------------------------------------------------------- GN step
def test_gn_step_closed_forms():
    psi, sing, cl = oracle.gn_step(np.eye(6), np.zeros(6))
    assert not sing and np.all(psi == 0)
    psi, sing, cl = oracle.gn_step(np.eye(6), np.eye(6)[0], damping_rel=0.0)
    np.testing.assert_array_equal(psi, -np.eye(6)[0])
    psi, sing, cl = oracle.gn_step(np.zeros((6, 6)), np.ones(6))
    assert sing
    psi, sing, cl = oracle.gn_step(np.eye(6) * 1e-3, np.ones(6), step_clamp=1.0)
    assert cl and abs(np.linalg.norm(psi) - 1.0) < 1e-14


def test_gn_step_solves_damped_system():
    g = np.random.default_rng(8)
    for _ in range(100):
        A = g.normal(size=(6, 6))
        H = A @ A.T + 1e-3 * np.eye(6)
        b = g.normal(size=6)
        psi, sing, cl = oracle.gn_step(H, b, damping_rel=1e-6, step_clamp=1e9)
        lam = 1e-6 * np.trace(H) / 6
        assert not sing and not cl
        assert np.linalg.norm((H + lam * np.eye(6)) @ psi + b) < 1e-9 * max(1, np.linalg.norm(b))


def test_gn_convergence_scan_vs_itself():
    """displaced by <= 0.2 (m, rad), iterated GN recovers < 1e-3."""
    m3, c6, r = _self_scene(r=1.0)
    cfg = oracle.make_config(voxel_resolution=r, loop_recency_gap=0, neighbor_count=1)
    kfs = oracle.Keyframes([(m3, c6)], [0.0], r)
    g = np.random.default_rng(9)
    n_ok = 0
    trials = 100
    poses = []
    for _ in range(trials):
        xi = g.normal(size=6)
        xi *= g.uniform(0.0, 0.2) / np.linalg.norm(xi)
        poses.append(synth.to12(expm(hat(xi))))
    pose = np.ascontiguousarray(np.stack(poses))
    kp = np.ascontiguousarray(np.tile(synth.to12(np.eye(4)), (trials, 1, 1)))
    for _ in range(20):
        oracle.particles(cfg, kfs, 1.0, pose, kp, m3, c6)
    for i in range(trials):
        T = T44(pose[i])
        ang = np.linalg.norm(Rotation.from_matrix(T[:3, :3]).as_rotvec())
        n_ok += (np.linalg.norm(T[:3, 3]) < 1e-3) and (ang < 1e-3)
    assert n_ok >= 99


# --------------------------------------------------------------------- neighbours / loop
def _kf_line(xs, cur_x, count, gap, K_pad=None):
    kfs_cloud = (np.zeros((1, 3), np.float32), np.array([[1, 0, 0, 1, 0, 1]], np.float32))
    K = len(xs)
    cfg = oracle.make_config(voxel_resolution=1.0, loop_recency_gap=gap, neighbor_count=count)
    kfs = oracle.Keyframes([kfs_cloud] * K, np.arange(K, dtype=float), 1.0)
    pose = synth.to12(synth.pose(t=(cur_x, 0, 0)))[None].copy()
    kp = synth.to12(np.stack([synth.pose(t=(x, 0, 0)) for x in xs]))[None].copy()
    return oracle.particles(cfg, kfs, float(K), pose, kp, np.zeros((1, 3)),
                            np.array([[1, 0, 0, 1, 0, 1]]), apply_update=False, slots=True)


def test_neighbours_nearest_ties_lower_and_gap_boundary():
    nb = GOLD["neighbours"]
    out = _kf_line(nb["kf_x"], nb["current_x"], nb["count"], gap=10)
    assert list(out["slot_kf"][0]) == nb["slots"]
    out = _kf_line([2.0, 0.0, 2.0, 5.0], 1.0, 3, gap=10)  # d = 1, 1, 1, 4: ties -> lower ids
    assert list(out["slot_kf"][0]) == [0, 1, 2]
    # latest = 3; gap 2: old <=> id <= 1 (inclusive); slots {2, 3} only -> no loop
    out = _kf_line([0.0, 0.0, 5.0, 5.0], 5.0, 2, gap=2)
    assert list(out["slot_kf"][0]) == [2, 3] and not (out["flags"][0] & 1)
    out = _kf_line([0.0, 5.0, 5.0, 9.0], 5.0, 2, gap=2)  # slot 1 = id 1 = latest - gap -> loop
    assert list(out["slot_kf"][0]) == [1, 2] and (out["flags"][0] & 1)
    out = _kf_line([0.0, 9.0], 0.0, 3, gap=10)  # K < 3 => min(3, K) slots
    assert list(out["slot_kf"][0]) == [0, 1, -1]


# --------------------------------------------------------------------- propagation
def test_propagation_ratio_hand_case():
    p = GOLD["propagation"]
    np.testing.assert_array_equal(oracle.propagation_ratio(p["D"], p["t_o"], p["D_now"]), p["r"])
    assert oracle.propagation_ratio([0.0, 1.0], 1, 1.0) is None  # zero denominator


def test_propagation_applies_scaled_twist_and_keeps_older_keyframes():
    """Eq.10: T_k <- T_k exp(r_k psi) for t_o <= k <= latest; older keyframes bit-identical."""
    s = synth.c1()
    m3, c6 = s.keyframes[0]
    K = 5
    cfg = oracle.make_config(voxel_resolution=s.r, loop_recency_gap=3, neighbor_count=3)
    # keyframes 0 and 4 far away (never neighbours); 1..3 near the scan's keyframe pose
    g = np.random.default_rng(10)
    base = s.kf_gt[0]
    kfT = [synth.pose(t=(60, 60, 0))]
    kfT += [base @ synth.pose(g.normal(0, 0.002, 3), g.normal(0, 0.02, 3)) for _ in range(3)]
    kfT += [base @ synth.pose(t=(30, 0, 0))]
    kfs = oracle.Keyframes([(m3, c6)] * K, [0.0, 1.0, 2.0, 3.0, 4.0], s.r)
    pose = synth.to12(s.T_gt @ synth.pose((0.01, 0, 0), (0.05, 0, 0)))[None].copy()
    kp0 = synth.to12(np.stack(kfT))[None].copy()
    kp = kp0.copy()
    out = oracle.particles(cfg, kfs, 5.0, pose, kp, s.scan_mean3, s.scan_cov6, slots=True)
    assert out["flags"][0] & 2
    t_o = out["slot_kf"][0].min()
    assert t_o == 1
    psi = out["psi6"][0]
    assert np.array_equal(kp[0, 0], kp0[0, 0])
    np.testing.assert_array_equal(kp[0, 1], kp0[0, 1])  # r = 0 at t_o
    for k in range(2, K):
        rk = (k - 1) / (5.0 - 1.0)
        ref = T44(kp0[0, k]) @ expm(hat(rk * psi))
        np.testing.assert_allclose(T44(kp[0, k])[:3], ref[:3], atol=2e-6)


# --------------------------------------------------------------------- weights, dead, respawn
def test_weights_closed_forms():
    wc = GOLD["weights_two"]
    _, e, w, m, S = oracle.weights(np.array(wc["L"]))
    np.testing.assert_allclose(w, wc["w"], rtol=1e-15)
    _, _, w, _, _ = oracle.weights(np.full(7, -123.0))
    np.testing.assert_array_equal(w, np.full(7, 1 / 7))
    L, _, w, _, _ = oracle.weights(np.zeros(5), np.array([-1.0, -2, -3, -4, -5]))
    np.testing.assert_array_equal(L, [-1.0, -2, -3, -4, -5])  # L += l (Eq.11 in logs)
    g = np.random.default_rng(11)
    _, _, w, _, _ = oracle.weights(g.normal(0, 300, 100_000))
    assert abs(w.sum() - 1) < 1e-12


def test_representative_cases():
    for c in GOLD["representative"]["cases"]:
        assert oracle.representative(np.array(c["w"])) == c["rep"]


def test_respawn_hand_case_boundary():
    rb = GOLD["respawn_boundary"]
    L, e, w, m, S = oracle.weights(np.zeros(3), np.array(rb["l"]))
    dead, nd = oracle.dead(np.array(rb["l"]), w)
    assert list(dead) == rb["dead"] and nd == 1
    q = [0 if dead[i] else math.floor(e[i] * 2**32) for i in range(3)]
    assert q == rb["q"] and sum(q) == rb["Q"]
    assert list(oracle.resample(e, dead, rb["U_last_donor0"])) == [-1, 0, -1]
    assert list(oracle.resample(e, dead, rb["U_first_donor2"])) == [-1, 2, -1]
    assert list(oracle.resample(e, dead, 0)) == [-1, 0, -1]
    assert list(oracle.resample(e, dead, 2**32 - 1)) == [-1, 2, -1]


def test_no_dead_no_change():
    e = np.array([1.0, 0.5, 0.25])
    assert list(oracle.resample(e, np.zeros(3, np.uint8), 12345)) == [-1, -1, -1]


def test_all_dead_is_degenerate():
    with pytest.raises(RuntimeError):
        oracle.resample(np.ones(3), np.ones(3, np.uint8), 7)


def _systematic_brute_force(e, dead, U):
    """Per-draw systematic search with exact rationals: p_r = (r + U/2^32) Q / D,
    donor_r = min{i : C_i > p_r}; the r-th dead slot (ascending) takes donor_r."""
    q = [0 if dead[i] else math.floor(e[i] * 2**32) for i in range(len(e))]
    C = np.cumsum(np.array(q, dtype=object))
    Q = int(C[-1])
    D = int(sum(dead))
    donors = []
    for r in range(D):
        p = (Fraction(r) + Fraction(U, 2**32)) * Fraction(Q, D)
        donors.append(next(i for i in range(len(e)) if C[i] > p))
    out = [-1] * len(e)
    it = iter(donors)
    for i in range(len(e)):
        if dead[i]:
            out[i] = next(it)
    return out, q, Q, D


def test_resample_equals_exact_systematic_search_and_count_invariants():
    g = np.random.default_rng(12)
    for trial in range(300):
        N = int(g.integers(1, 60))
        e = np.exp(-g.exponential(3.0, N))
        e[g.integers(0, N)] = 1.0
        dead = (g.random(N) < g.uniform(0, 0.9)).astype(np.uint8)
        if dead.all():
            dead[g.integers(0, N)] = 0
        U = int(g.integers(0, 2**32))
        donor = oracle.resample(e, dead, U)
        ref, q, Q, D = _systematic_brute_force(e, dead, U)
        assert list(donor) == ref
        copies = np.bincount(donor[donor >= 0], minlength=N)
        assert copies.sum() == D
        for i in range(N):
            lo, hi = (D * q[i]) // Q, -((-D * q[i]) // Q)
            assert lo <= copies[i] <= hi
        assert np.all(donor[dead == 0] == -1)
        assert np.all(dead[donor[donor >= 0]] == 0)


def test_resample_statistics_uniform_survivors():
    """N = 4, one dead, uniform survivors: each survivor donates w.p. 1/3 (3 sigma)."""
    g = np.random.default_rng(13)
    e = np.ones(4)
    dead = np.array([0, 0, 1, 0], np.uint8)
    n = 10_000
    counts = np.zeros(4)
    for U in g.integers(0, 2**32, n):
        counts[oracle.resample(e, dead, int(U))[2]] += 1
    p = 1 / 3
    sd = math.sqrt(n * p * (1 - p))
    for i in (0, 1, 3):
        assert abs(counts[i] - n * p) < 3 * sd
    assert counts[2] == 0


def test_full_update_invariants():
    s = synth.c1()
    cfg = oracle.make_config(voxel_resolution=s.r, loop_recency_gap=s.gap)
    kfs = oracle.Keyframes(s.keyframes, s.D, s.r)
    pose, kp, L = s.pose12.copy(), s.kf_pose12.copy(), np.zeros(s.N)
    out = oracle.update(cfg, kfs, s.D_now, pose, kp, L, s.scan_mean3, s.scan_cov6, s.U)
    assert out["status"] == 0
    assert abs(out["weight"].sum() - 1) < 1e-12
    d = out["donor"]
    assert out["n_dead"] == (d >= 0).sum() == ((out["flags"] & 8) > 0).sum()
    for i in np.nonzero(d >= 0)[0]:
        assert np.array_equal(pose[i], pose[d[i]]) and L[i] == L[d[i]]
    assert out["representative"] == int(np.argmax(out["weight"]))


def test_resample_exact_ladder_boundaries():
    """Draws landing exactly on a rung boundary (p_r == C_i) go to the NEXT survivor
    (donor = min{i : C_i > p_r}); exercises the exact-division branch of the count formula."""
    for N, dead_idx, U in ((3, [2], 2**31), (5, [1, 3], 0), (6, [0, 5], 2**31), (4, [3], 0)):
        e = np.ones(N)
        dead = np.zeros(N, np.uint8)
        dead[dead_idx] = 1
        ref, *_ = _systematic_brute_force(e, dead, U)
        assert list(oracle.resample(e, dead, U)) == ref


def test_sandwich_rotates_the_scan_covariance_eigenvectors():
    """C = Sigma' + R Sigma R^T (Eq.4): with Sigma' = eps I and a residual along the rotated
    eigenvector R u_i of Sigma, l = -s^2 / (eps + lambda_i) for every rotation R — a transposed
    or missing R in the sandwich gives another value (spectral theorem; not the oracle's own
    formula)."""
    g = np.random.default_rng(7)
    eps, s = 0.01, 0.05
    lam = np.array([0.09, 0.04, 0.002])
    U = Rotation.from_rotvec(g.normal(size=3)).as_matrix()
    Sig = U @ np.diag(lam) @ U.T
    c6 = np.array([[Sig[0, 0], Sig[0, 1], Sig[0, 2], Sig[1, 1], Sig[1, 2], Sig[2, 2]]],
                  np.float32)
    Sig = np.array([[c6[0, 0], c6[0, 1], c6[0, 2]], [c6[0, 1], c6[0, 3], c6[0, 4]],
                    [c6[0, 2], c6[0, 4], c6[0, 5]]], np.float64)  # the fp32-rounded input
    lam, U = np.linalg.eigh(Sig)
    mu_p = np.array([[1.0, 1.0, 1.0]], np.float32)  # middle of voxel (0, 0, 0) at r = 2
    m = oracle.Map(mu_p, np.array([[eps, 0, 0, eps, 0, eps]], np.float32), 2.0)
    mu = np.array([[0.3, -0.2, 0.1]], np.float32)
    for trial in range(4):
        R = Rotation.from_rotvec(g.normal(size=3) * 0.7).as_matrix()
        for i in range(3):
            v = s * (R @ U[:, i])              # wanted residual e = mu' - (R mu + t)
            t = mu_p[0] - R @ mu[0] - v
            T = np.eye(4)
            T[:3, :3], T[:3, 3] = R, t
            rel32 = np.asarray(T[:3, :4], np.float32)
            res = oracle.pair_linearize(m, mu, c6, rel32, T[:3, :4])
            assert res.n == 1
            e = mu_p[0].astype(np.float64) - (R @ mu[0].astype(np.float64) + t)
            expect = -(e @ e) / (eps + lam[i])  # e is v up to fp32 input rounding
            assert res.l == pytest.approx(expect, rel=1e-6), (trial, i)
