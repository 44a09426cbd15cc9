"""Edge cases of the CUDA path against the oracle: scan sizes at and around the
shared-memory stages (256 points general, 448 plane-form) and the 4-point probe batch (1, 2,
3, 5, 255, 256, 257, 447, 448, 449, 513, 897), every
neighbour count 1..MCS_MAX_NEIGHBORS, GN over all slots, a voxel size of 2 m, and one-point
keyframes."""
import dataclasses

import numpy as np
import pytest

import oracle
import paper_2504_18056_b200 as mcs
import synth
from test_gpu_parity import (G_RTOL, H_RTOL, L_RTOL, ROT_TOL, T_TOL, check_slots, make_ctx,
                             orc_cfg, pose_err, rel_err)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2s():
    return synth.subset(synth.c2(N=2000), 1500)


# The north-star tolerances are for whole scans.  With a handful of points the fp32 rounding of
# q (~1e-6 m at 10-20 m) against centimetre residuals is ~1e-4 of e per point and nothing
# averages it out: l is then compared at 2e-3 relative, g at 1e-2, H at the full 1e-3, and the
# (rank-deficient, damping-dominated) pose step is not compared.  mcs.h states this S >= 64
# domain of the 1e-4 contract.
FEW = 64


def _eval_parity(s, **kw):
    with make_ctx(s, **kw) as ctx:
        g = ctx.eval(s.scan_mean3, s.scan_cov6)
        g["nonplanar"] = ctx.scan_nonplanar()
    o = oracle.particles(orc_cfg(s, **kw), oracle.Keyframes(s.keyframes, s.D, s.r), s.D_now,
                         s.pose12.copy(), s.kf_pose12.copy(), s.scan_mean3, s.scan_cov6,
                         apply_update=False, slots=True)
    if s.S >= FEW:
        check_slots(g, o, s.S)
    else:
        np.testing.assert_array_equal(g["slot_kf"], o["slot_kf"])
        np.testing.assert_array_equal(g["slot_n"], o["slot_n"])
        assert np.all(np.abs(g["slot_loglik"] - o["slot_l"]) <= 2e-3 * np.abs(o["slot_l"]) + 1e-6)
    return g, o


def _update_parity(s, **kw):
    nd = dict(posterior_floor=0.0, loglik_rel_floor=-np.inf)
    with make_ctx(s, **kw, **nd) as ctx:
        g = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        st = ctx.get_particles()
    pose, kp, L = s.pose12.copy(), s.kf_pose12.copy(), np.zeros(s.N)
    o = oracle.update(orc_cfg(s, **kw, **nd), oracle.Keyframes(s.keyframes, s.D, s.r),
                      s.D_now, pose, kp, L, s.scan_mean3, s.scan_cov6, s.U)
    if s.S >= FEW:  # the north-star contract: 1e-4 relative, no absolute slack
        assert np.all(np.abs(g["loglik"] - o["loglik"]) <= L_RTOL * np.abs(o["loglik"]))
    else:
        assert np.all(np.abs(g["loglik"] - o["loglik"]) <= 2e-3 * np.abs(o["loglik"]) + 1e-6)
    np.testing.assert_array_equal(g["flags"] & 1, o["flags"] & 1)
    if s.S < FEW:
        # g = -2 sum J^T Omega e inherits the ~1e-4-per-point rounding of e, with cancellation
        # across a handful of terms: 1e-2; H depends on e only through the correspondences (and
        # on m = q - t, relative 1e-7): the full 1e-3.  Zero rows stay exactly zero.
        gn = np.linalg.norm(o["grad6"], axis=1) > 0
        assert np.all(rel_err(g["grad6"][gn], o["grad6"][gn], axis=1) <= 1e-2)
        assert not g["grad6"][~gn].any()
        Hg = mcs.unpack_h21(g["hess21"]).reshape(-1, 36).astype(float)
        Ho = o["hess36"].reshape(-1, 36)
        hz = np.linalg.norm(Ho, axis=1) > 0
        assert np.all(rel_err(Hg[hz], Ho[hz], axis=1) <= H_RTOL)
        return g, o
    gn = np.linalg.norm(o["grad6"], axis=1) > 0
    assert np.all(rel_err(g["grad6"][gn], o["grad6"][gn], axis=1) <= G_RTOL)
    assert not g["grad6"][~gn].any()
    np.testing.assert_array_equal(g["flags"], o["flags"])
    ang, dt = pose_err(st["pose12"], pose)
    assert ang.max() <= ROT_TOL and dt.max() <= T_TOL, (ang.max(), dt.max())
    ak, dk = pose_err(st["kf_pose12"].reshape(-1, 12), kp.reshape(-1, 12))
    assert ak.max() <= ROT_TOL and dk.max() <= T_TOL
    return g, o


@pytest.mark.parametrize("S", [1, 2, 3, 5, 255, 256, 257, 447, 448, 449, 513, 897])
def test_scan_sizes_around_stage_and_batch(c2s, S):
    s = dataclasses.replace(c2s, scan_mean3=np.ascontiguousarray(c2s.scan_mean3[:S]),
                            scan_cov6=np.ascontiguousarray(c2s.scan_cov6[:S]))
    _eval_parity(s)
    _update_parity(s)


@pytest.mark.parametrize("nb", [1, 2, 3, 4])  # 1..MCS_MAX_NEIGHBORS
def test_every_neighbour_count(c2s, nb):
    _eval_parity(c2s, neighbor_count=nb)
    _update_parity(c2s, neighbor_count=nb)


def test_gn_over_all_slots(c2s):
    g, o = _update_parity(c2s, gn_slots=1)
    assert (o["flags"] & 2).mean() > 0.5


def test_voxel_size_two_metres():
    s = synth.c1()
    m3, c6 = s.keyframes[0]
    s2 = dataclasses.replace(s, r=2.0, pose12=np.ascontiguousarray(s.pose12[:400]),
                             kf_pose12=np.ascontiguousarray(s.kf_pose12[:400]))
    _eval_parity(s2)
    _update_parity(s2)


def test_one_point_keyframes():
    """Keyframes of a single Gaussian: a one-cell table; most points miss, the rest match it."""
    s = synth.c1()
    m3, c6 = s.keyframes[0]
    kfs = [(m3[i:i + 1].copy(), c6[i:i + 1].copy()) for i in (0, 100, 900)]
    kp = np.ascontiguousarray(np.repeat(s.kf_pose12[:300], 3, axis=1))
    s2 = dataclasses.replace(s, keyframes=kfs, D=np.array([0.0, 1.0, 2.0]),
                             pose12=np.ascontiguousarray(s.pose12[:300]), kf_pose12=kp)
    g, o = _eval_parity(s2)
    assert g["slot_n"].max() <= s2.S


def test_far_from_origin_correspondences_stay_exact():
    """R27 pins the fp32 key path (relative pose entries, transform, floor), so even 400 km
    from the origin, where fp32 poses carry ~3 cm of rounding and l is no longer comparable
    (the tolerances assume scenes within +-50 m), the GPU and the oracle pick the same cells:
    slot keyframes and match counts agree exactly."""
    s = synth.c1()
    off = np.array([4.0e5, -3.0e5, 120.0], np.float32)
    P = s.pose12.reshape(-1, 3, 4).copy()
    P[:, :, 3] += off
    K = s.kf_pose12.reshape(s.N, -1, 3, 4).copy()
    K[:, :, :, 3] += off
    s2 = dataclasses.replace(s, pose12=np.ascontiguousarray(P.reshape(-1, 12)),
                             kf_pose12=np.ascontiguousarray(K.reshape(s.N, -1, 12)))
    with make_ctx(s2) as ctx:
        g = ctx.eval(s2.scan_mean3, s2.scan_cov6)
    o = oracle.particles(orc_cfg(s2), oracle.Keyframes(s2.keyframes, s2.D, s2.r), s2.D_now,
                         s2.pose12.copy(), s2.kf_pose12.copy(), s2.scan_mean3, s2.scan_cov6,
                         apply_update=False, slots=True)
    np.testing.assert_array_equal(g["slot_kf"], o["slot_kf"])
    np.testing.assert_array_equal(g["slot_n"], o["slot_n"])
    assert g["slot_n"].sum() > 0


def test_keyframe_larger_than_the_sparse_table_budget():
    """A keyframe of ~300k occupied cells: 4 x cells already exceeds the 64 MiB table budget, so
    its table stays at the minimum capacity (load up to 1/4, linear-probing chains common)
    instead of the sparse 1/64; correspondences and l still match the oracle."""
    s = synth.c1()
    m3, c6 = s.keyframes[0]
    g = np.stack(np.meshgrid(np.arange(70), np.arange(70), np.arange(62), indexing="ij"), -1)
    fill = (g.reshape(-1, 3) * 0.5 + 0.25 + np.array([40.0, -20.0, -10.0])).astype(np.float32)
    fc = np.tile(np.array([1e-2, 0, 0, 1e-2, 0, 1e-2], np.float32), (len(fill), 1))
    big = (np.concatenate([m3, fill]), np.concatenate([c6, fc]))
    s2 = dataclasses.replace(s, keyframes=[big], pose12=np.ascontiguousarray(s.pose12[:300]),
                             kf_pose12=np.ascontiguousarray(s.kf_pose12[:300]))
    assert len(big[0]) > 300_000
    _eval_parity(s2)


@pytest.mark.parametrize("corr", ["cell", "nn27"])
def test_table_budget_does_not_change_results(c2s, corr):
    """mcs_config.kf_table_mib only changes where cells sit in the table (minimum load-1/4
    capacity with 0, up to 64 slots per cell by default): every output is bitwise equal."""
    kw = dict(corr_mode=mcs.CORR_NN27, nn_radius=c2s.r) if corr == "nn27" else {}
    s = synth.subset(c2s, 300) if corr == "nn27" else c2s
    outs = []
    for mib in (0, 64):
        with make_ctx(s, kf_table_mib=mib, **kw) as ctx:
            ev = ctx.eval(s.scan_mean3, s.scan_cov6)
            up = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        outs.append((ev, up))
    (e0, u0), (e1, u1) = outs
    for k in e0:
        np.testing.assert_array_equal(e0[k], e1[k], err_msg=k)
    for k in ("loglik", "grad6", "hess21", "psi6", "weight", "donor", "flags"):
        np.testing.assert_array_equal(u0[k], u1[k], err_msg=k)
    assert u0["representative"] == u1["representative"]


def test_combine_shapes_agree_bitwise():
    """a3 runs one thread per particle from 40,000 particles up and one thread per (slot,
    particle) below (MCS_COMBINE_SLOTS_BELOW): both sum the slots in the same order, so the
    per-particle outputs of the same particles agree bitwise across the two shapes."""
    s = synth.c2(N=40000)
    nd = dict(posterior_floor=0.0, loglik_rel_floor=-np.inf)
    res = []
    for n in (40000, 39999):
        sub = synth.subset(s, n)
        with make_ctx(sub, **nd) as ctx:
            g = ctx.update(sub.scan_mean3, sub.scan_cov6, sub.D_now, sub.U)
            st = ctx.get_particles()
        res.append((g, st))
    (g0, s0), (g1, s1) = res
    for k in ("loglik", "grad6", "hess21", "psi6", "flags"):
        np.testing.assert_array_equal(g0[k][:39999], g1[k], err_msg=k)
    np.testing.assert_array_equal(s0["pose12"][:39999], s1["pose12"])
    np.testing.assert_array_equal(s0["kf_pose12"][:39999], s1["kf_pose12"])


def test_keyframe_bbox_extent_limit():
    """mcs.h: a keyframe's occupied cells must fit 2046 x 2047 x 1023 cells (the 32-bit
    bbox-local table keys); one cell more on any axis is MCS_E_INVALID_ARG with no keyframe
    added, exactly the limit is accepted."""
    r = 0.5
    cov = np.tile(np.array([0.5, 0, 0, 0.5, 0, 0.5], np.float32), (2, 1))
    with mcs.Context(4, 4, 8, voxel_resolution=r) as ctx:
        for axis, cells in ((0, 2046), (1, 2047), (2, 1023)):
            for extra, ok in ((0, True), (1, False)):
                m = np.zeros((2, 3), np.float32)
                m[1, axis] = (cells - 1 + extra) * r + 0.1  # cells 0 .. cells - 1 + extra
                before = ctx.sizes[1]
                if ok:
                    ctx.add_keyframe(m, cov, float(before))
                    assert ctx.sizes[1] == before + 1
                else:
                    with pytest.raises(mcs.MCSError) as ei:
                        ctx.add_keyframe(m, cov, float(before))
                    assert ei.value.status == 1 and ctx.sizes[1] == before


def _cov6_from_eig(rng, lam):
    """fp32 cov6 (xx, xy, xz, yy, yz, zz) of V diag(lam) V^T, V random rotations (fp64)."""
    V, _ = np.linalg.qr(rng.standard_normal((len(lam), 3, 3)))
    A = np.einsum("nij,nj,nkj->nik", V, lam, V)
    return np.ascontiguousarray(A[:, [0, 0, 0, 1, 1, 2], [0, 1, 2, 1, 2, 2]].astype(np.float32))


def test_plane_form_scan_takes_the_plane_path(c2s):
    """The synthetic scans are GICP plane-regularised (eigenvalues (1, 1, 1e-3), R9): every
    point is plane-form, so the sweep's plane instantiation runs (R36) — parity as usual."""
    g, _ = _eval_parity(c2s)
    assert g["nonplanar"] == 0


def test_general_scan_covariances(c2s):
    """Random SPD scan covariances (three distinct eigenvalues, log-uniform in [1e-3, 1]):
    the general instantiation (Sigma = lam3 I + u u^T + v v^T) against the oracle."""
    rng = np.random.default_rng(36)
    lam = np.exp(rng.uniform(np.log(1e-3), 0.0, (c2s.S, 3)))
    s = dataclasses.replace(c2s, scan_cov6=_cov6_from_eig(rng, lam))
    g, _ = _eval_parity(s)
    assert g["nonplanar"] == s.S
    _update_parity(s)


def test_one_general_point_selects_the_general_path(c2s):
    """A single non-plane point sends the whole scan through the general instantiation."""
    rng = np.random.default_rng(7)
    c6 = c2s.scan_cov6.copy()
    c6[17] = _cov6_from_eig(rng, np.array([[0.7, 0.3, 2e-3]]))[0]
    s = dataclasses.replace(c2s, scan_cov6=c6)
    g, _ = _eval_parity(s)
    assert g["nonplanar"] == 1
    _update_parity(s)


@pytest.mark.parametrize("split,plane", [(1e-7, True), (2e-6, False)])
def test_plane_merge_tolerance(c2s, split, plane):
    """R36's merge rule: top-two eigenvalue splits within 2^-21 of the largest (4 ulps, the
    rounding of the fp32 entries) are plane-form (their mean is used), larger ones are not;
    both sides of the rule agree with the oracle, which uses the covariance as given."""
    rng = np.random.default_rng(11)
    lam = np.tile([1.0 + split, 1.0, 1e-3], (c2s.S, 1))
    s = dataclasses.replace(c2s, scan_cov6=_cov6_from_eig(rng, lam))
    g, _ = _eval_parity(s)
    assert (g["nonplanar"] == 0) == plane, g["nonplanar"]
    _update_parity(s)
