"""Pins for the oracle's NEXT rows: Philox4x32-10 + Box-Muller noise, the
prediction step (Eq.1) with the elevator vertical walk, the keyframe-insertion
overlap test, and the multi-iteration / post-update weighting variants (R12, R13)."""
import json
import os

import numpy as np
import pytest
from scipy.linalg import expm
from scipy.stats import chi2

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def T44(T12):
    T = np.eye(4)
    T[:3, :4] = np.asarray(T12, float).reshape(3, 4)
    return T


def test_philox_known_answers():
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for c in kat["cases"]:
        ctr = [int(x, 16) for x in c["ctr"]]
        key = [int(x, 16) for x in c["key"]]
        assert [int(v) for v in oracle.philox4x32_10(ctr, key)] == [int(x, 16) for x in c["out"]]


def test_normals_are_standard_normal():
    z = np.stack([oracle.normals8(7, 3, g) for g in range(40_000)])
    assert np.all(np.isfinite(z))
    n = len(z)
    assert np.all(np.abs(z.mean(0)) < 5 / np.sqrt(n))
    assert np.all(np.abs(z.var(0) - 1) < 5 * np.sqrt(2 / n))
    c = np.corrcoef(z.T)
    assert np.abs(c - np.eye(8)).max() < 5 / np.sqrt(n)
    # different frames / seeds give different streams
    assert not np.array_equal(oracle.normals8(7, 3, 0), oracle.normals8(7, 4, 0))
    assert not np.array_equal(oracle.normals8(7, 3, 0), oracle.normals8(8, 3, 0))


def test_predict_zero_noise_is_composition():
    g = np.random.default_rng(1)
    P = synth.to12(np.stack([synth.pose(g.normal(size=3), g.uniform(-30, 30, 3))
                             for _ in range(50)]))
    dT = synth.pose((0.01, -0.02, 0.1), (0.5, 0.1, 0.0))
    out = P.copy()
    oracle.predict(out, synth.to12(dT), np.zeros((6, 6)), seed=1, frame=0)
    for i in range(50):
        ref = T44(P[i]) @ T44(synth.to12(dT))
        np.testing.assert_allclose(T44(out[i]), ref, atol=3e-6)


def test_predict_noise_has_the_odometry_covariance():
    """Eq.1: delta ~ N(0, Sigma) in the tangent space of dT; recovered by the pinned SE(3) log."""
    N = 20_000
    A = np.random.default_rng(2).normal(size=(6, 6)) * 0.02
    cov = A @ A.T + np.diag([1e-4] * 3 + [1e-5] * 3)
    P = np.tile(synth.to12(np.eye(4)), (N, 1))
    dT = synth.pose((0.0, 0.0, 0.2), (1.0, 0.0, 0.0))
    oracle.predict(P, synth.to12(dT), cov, seed=11, frame=5)
    inv = np.linalg.inv(T44(synth.to12(dT)))
    d = np.stack([oracle.se3_log((inv @ T44(P[i]))[:3]) for i in range(N)])
    emp = np.cov(d.T)
    # every quadratic form matches within ~5 sigma of its sampling error
    for v in np.eye(6):
        sd = np.sqrt(2 / N) * (v @ cov @ v)
        assert abs(v @ emp @ v - v @ cov @ v) < 6 * sd + 1e-9
    assert np.all(np.abs(d.mean(0)) < 6 * np.sqrt(np.diag(cov) / N))
    # Mahalanobis distances are chi^2(6)
    m2 = np.einsum("ni,ij,nj->n", d, np.linalg.inv(cov), d)
    assert abs(np.mean(m2 < chi2.ppf(0.9, 6)) - 0.9) < 0.01


def test_predict_vertical_walk_only_moves_z():
    N = 20_000
    P = np.tile(synth.to12(synth.pose((0.1, 0.2, 0.3), (1, 2, 3))), (N, 1))
    P0 = P.copy()
    oracle.predict(P, synth.to12(np.eye(4)), np.zeros((6, 6)), seed=3, frame=1,
                   vertical_sigma=2.0)
    dz = P[:, 11].astype(float) - P0[:, 11]
    assert np.abs(P[:, [3, 7]] - P0[:, [3, 7]]).max() < 1e-6
    assert abs(dz.std() - 2.0) < 0.05 and abs(dz.mean()) < 0.05


def test_predict_rejects_indefinite_covariance():
    P = np.tile(synth.to12(np.eye(4)), (2, 1))
    with pytest.raises(ValueError):
        oracle.predict(P, synth.to12(np.eye(4)), -np.eye(6), 1, 1)


def test_overlap_pins():
    s = synth.c1()
    m3, c6 = s.keyframes[0]
    m = oracle.Map(m3, c6, s.r)
    I = synth.to12(np.eye(4))
    assert oracle.overlap(m, m3, I) == 1.0                       # scan vs its own map
    far = synth.to12(synth.pose(t=(1000.0, 0, 0)))
    assert oracle.overlap(m, m3, far) == 0.0
    # brute force: fraction of transformed points whose fp32 cell is an occupied cell
    rel = synth.to12(synth.pose((0.0, 0.0, 0.05), (0.3, -0.2, 0.0)))
    R, t = rel.reshape(3, 4)[:, :3], rel.reshape(3, 4)[:, 3]
    q = np.empty_like(s.scan_mean3)
    for a in range(3):  # fmaf chain in float64 is exact here? no: use the oracle's cell_of pin
        q[:, a] = (s.scan_mean3.astype(np.float64) @ R[a].astype(np.float64) + t[a])
    cells = {tuple(c) for c in np.floor(m3 * np.float32(1 / s.r)).astype(np.int64)}
    qc = np.floor(q.astype(np.float32) * np.float32(1 / s.r)).astype(np.int64)
    bf = np.mean([tuple(c) in cells for c in qc])
    assert abs(oracle.overlap(m, s.scan_mean3, rel) - bf) <= 3 / len(q)  # face-rounding slack


def test_iterations_and_post_update_weighting():
    s = synth.c1()
    kfs = oracle.Keyframes(s.keyframes, s.D, s.r)
    base = dict(voxel_resolution=s.r, loop_recency_gap=s.gap, posterior_floor=0.0,
                loglik_rel_floor=-np.inf)

    def run(**kw):
        pose, kp, L = s.pose12.copy(), s.kf_pose12.copy(), np.zeros(s.N)
        out = oracle.update(oracle.make_config(**base, **kw), kfs, s.D_now, pose, kp, L,
                            s.scan_mean3, s.scan_cov6, s.U)
        return out, pose

    o1, p1 = run()
    o1b, _ = run(gn_iterations=1, weight_after_update=0)
    assert np.array_equal(o1["loglik"], o1b["loglik"])
    o3, p3 = run(gn_iterations=3)
    np.testing.assert_array_equal(o3["loglik"], o1["loglik"])  # weighting l is pre-update (R13)
    terr = lambda P: np.linalg.norm(P.reshape(-1, 3, 4)[:, :, 3] - s.T_gt[:3, 3], axis=1)
    assert np.median(terr(p3)) < np.median(terr(p1)) < np.median(terr(s.pose12))
    o3p, p3p = run(gn_iterations=3, weight_after_update=1)
    np.testing.assert_array_equal(p3p, p3)
    assert np.median(o3p["loglik"]) > np.median(o1["loglik"])  # GN ascent improved l


# ------------------------------------------------------------------ NN27 correspondence (R33)
from fractions import Fraction


def _f32_round(x: Fraction) -> np.float32:
    """x correctly rounded to fp32 (ties to even), independent of the oracle's arithmetic."""
    f = np.float32(float(x))
    cands = [np.nextafter(f, np.float32(-np.inf)), f, np.nextafter(f, np.float32(np.inf))]
    best = None
    for c in cands:
        d = abs(Fraction(float(c)) - x)
        key = (d, int(np.array(c, np.float32).view(np.uint32)) & 1)
        if best is None or key < best[0]:
            best = (key, c)
    return np.float32(best[1])


def _fmaf(a, b, c):
    return _f32_round(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def _brute_nn(q, means32, cells, r, nn_radius):
    """Nearest representative over ALL cells within nn_radius, pinned fp32 d2 (exact fma)."""
    q = np.asarray(q, np.float32)
    r2 = np.float32(nn_radius) * np.float32(nn_radius)
    d = (means32 - q).astype(np.float32)
    approx = (d.astype(np.float64) ** 2).sum(1)
    qc = np.floor(q * np.float32(1.0 / r)).astype(np.int64)
    best = None
    for k in np.nonzero(approx <= float(r2) * 1.001 + 1e-12)[0]:
        dx, dy, dz = d[k]
        d2 = _fmaf(dz, dz, _fmaf(dy, dy, np.float32(dx * dx)))
        if not d2 <= r2:
            continue
        o = cells[k] - qc
        idx = int((o[2] + 1) * 9 + (o[1] + 1) * 3 + (o[0] + 1)) if np.abs(o).max() <= 1 else 99
        key = (float(d2), idx)
        if best is None or key < best[0]:
            best = (key, k)
    return -1 if best is None else int(best[1])


@pytest.mark.parametrize("nn_radius", [0.5, 0.3])
def test_nn27_is_the_bruteforce_nearest_neighbour(nn_radius):
    g = np.random.default_rng(11)
    r = 0.5
    pts = g.uniform(-1.5, 1.5, (500, 3)).astype(np.float32)
    cov = np.tile(np.array([0.01, 0, 0, 0.01, 0, 0.01], np.float32), (len(pts), 1))
    m = oracle.Map(pts, cov, r)
    n = len(m)
    means, _ = m.cells(np.arange(n))
    means32 = means.astype(np.float32)
    cells = np.array([oracle.cell_of(mu, r) for mu in means32], np.int64)
    m.set_corr(oracle.CORR_NN27, nn_radius)
    qs = g.uniform(-1.8, 1.8, (300, 3)).astype(np.float32)
    got = np.array([m.correspond(q) for q in qs])
    ref = np.array([_brute_nn(q, means32, cells, r, nn_radius) for q in qs])
    np.testing.assert_array_equal(got, ref)
    assert (got >= 0).mean() > 0.3
    # CELL is a different rule: it misses queries whose own voxel is empty
    m.set_corr(oracle.CORR_CELL)
    cell = np.array([m.correspond(q) for q in qs])
    assert ((cell < 0) & (got >= 0)).any()


def test_nn27_hand_case_across_a_face():
    r = 0.5
    m = oracle.Map(np.array([[0.49, 0.0, 0.0]], np.float32),
                   np.array([[0.25, 0, 0, 0.25, 0, 0.25]], np.float32), r)
    q = np.array([0.51, 0.0, 0.0], np.float32)  # next voxel along x, 0.02 m away
    assert m.correspond(q) == -1                  # CELL: empty voxel
    m.set_corr(oracle.CORR_NN27, 0.5)
    assert m.correspond(q) == 0
    m.set_corr(oracle.CORR_NN27, 0.01)           # outside the radius
    assert m.correspond(q) == -1
    # ties: two representatives at the same fp32 distance -> the lower (oz, oy, ox) index wins
    m2 = oracle.Map(np.array([[0.25, 0.25, -0.25], [0.25, 0.25, 0.75]], np.float32),
                    np.tile(np.array([0.25, 0, 0, 0.25, 0, 0.25], np.float32), (2, 1)), r)
    m2.set_corr(oracle.CORR_NN27, 0.5)
    k = m2.correspond(np.array([0.25, 0.25, 0.25], np.float32))
    means, _ = m2.cells([k])
    assert means[0][2] == np.float32(-0.25)      # oz = -1 comes first


def test_nn27_self_match_is_exact():
    """Scan = keyframe cloud with one point per cell, identity pose: every point matches its own
    cell at d2 = 0, so l = 0, b = 0 exactly, as under CELL."""
    s = synth.c1()
    m3, c6 = s.keyframes[0]
    m = oracle.Map(m3, c6, s.r)
    m.set_corr(oracle.CORR_NN27, s.r)
    r32, r64 = oracle.relpose(synth.to12(np.eye(4)), synth.to12(np.eye(4)))
    res = oracle.pair_linearize(m, m3, c6, r32, r64)
    assert res.n == len(m3) and res.l == 0.0 and np.all(res.b == 0.0)
    m.set_corr(oracle.CORR_CELL)
    res_c = oracle.pair_linearize(m, m3, c6, r32, r64)
    np.testing.assert_array_equal(res.corr, res_c.corr)


# ------------------------------------------------------------------ weight-splitting clones (R34)
def test_clone_split_shares_the_donor_weight():
    s = synth.c1()
    kfs = oracle.Keyframes(s.keyframes, s.D, s.r)

    def run(split):
        pose, kp, L = s.pose12.copy(), s.kf_pose12.copy(), np.zeros(s.N)
        out = oracle.update(oracle.make_config(voxel_resolution=s.r, loop_recency_gap=s.gap,
                                               clone_split=split), kfs, s.D_now, pose, kp, L,
                            s.scan_mean3, s.scan_cov6, s.U)
        return out, L

    oc, Lc = run(0)
    os_, Ls = run(1)
    np.testing.assert_array_equal(oc["donor"], os_["donor"])  # same e, dead set and U
    assert 0 < oc["n_dead"] < s.N
    donor = oc["donor"]
    copies = np.bincount(donor[donor >= 0], minlength=s.N)
    src = np.where(donor >= 0, donor, np.arange(s.N))  # whose L each slot holds
    expect = Lc - np.log1p(copies[src])                 # donor and each clone: L - ln(1 + c)
    np.testing.assert_allclose(Ls, expect, rtol=0, atol=1e-12)
    assert abs(os_["weight"].sum() - 1) < 1e-12
    # the split conserves each donor family's total weight before renormalisation
    fam = np.exp(Ls - Ls.max())
    for d in np.unique(donor[donor >= 0])[:20]:
        members = (src == d)
        assert np.isclose(fam[members].sum(), np.exp(Lc[d] - Ls.max()), rtol=1e-12)
