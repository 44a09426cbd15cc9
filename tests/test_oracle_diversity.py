"""Pins of the neighbour-particle diversity term (reading R35, flag `diversity_weight`).

The paper cites SVGD / GN-SVGD for "preserving sample diversity through neighbor particle
information" but its own update (Eqs.5-10) defines no such term; R35 takes
SVGD's kernel-gradient (repulsive) term with an RBF kernel on the current-pose translations:
    d_i = (2 / (h N)) sum_j (t_i - t_j) exp(-|t_i - t_j|^2 / h) = -grad_{t_i} (1/N) sum_j k(t_i, t_j)
and moves every translation by eta d_i after the GN step.  Pinned here by what the definition
fixes independently of its implementation: the gradient identity (central differences of the
kernel density), antisymmetry (sum_i d_i = 0), the closed form of a pair, vanishing limits
(N = 1, h -> 0, far particles), and eta = 0 / h -> 0 reducing the whole update to the plain one
bit for bit.  CPU only.
"""
import numpy as np
import pytest

import oracle
import synth


def test_pair_closed_form_and_antisymmetry():
    h = 0.5
    delta = np.array([0.3, -0.2, 0.1])
    t = np.stack([np.zeros(3), -delta])  # t_1 - t_2 = delta
    d = oracle.diversity(t, h)
    expect = delta / h * np.exp(-delta @ delta / h)  # (2 / (2h)) delta exp(-|delta|^2 / h)
    np.testing.assert_allclose(d[0], expect, rtol=1e-15)
    np.testing.assert_array_equal(d[1], -d[0])


def test_gradient_of_the_kernel_density():
    """d_i = -grad_{t_i} E_i, E_i = (1/N) sum_j exp(-|t_i - t_j|^2 / h): central differences."""
    g = np.random.default_rng(3)
    t = g.normal(0, 0.4, (7, 3))
    h = 0.3
    d = oracle.diversity(t, h)

    def E(i, ti):
        return np.mean(np.exp(-np.sum((ti - t) ** 2, axis=1) / h))

    eps = 1e-6
    for i in range(len(t)):
        grad = np.zeros(3)
        for c in range(3):
            tp, tm = t[i].copy(), t[i].copy()
            tp[c] += eps
            tm[c] -= eps
            # (the j = i term is exp(-eps^2 / h) at both tp and tm: it cancels)
            grad[c] = (E(i, tp) - E(i, tm)) / (2 * eps)
        np.testing.assert_allclose(d[i], -grad, rtol=1e-6, atol=1e-10)


def test_sum_vanishes_and_limits():
    g = np.random.default_rng(4)
    t = g.normal(0, 1.0, (50, 3))
    d = oracle.diversity(t, 0.7)
    np.testing.assert_allclose(d.sum(axis=0), 0.0, atol=1e-13)  # pairwise terms cancel
    assert not oracle.diversity(t[:1], 0.7).any()                # N = 1
    assert not oracle.diversity(t, 1e-300).any()                 # h -> 0: distinct particles decouple
    far = np.stack([np.zeros(3), np.array([1e3, 0, 0])])
    assert not oracle.diversity(far, 1.0).any()                  # exp underflows: no interaction


@pytest.mark.parametrize("kw", [dict(diversity_weight=0.0, diversity_bandwidth=0.5),
                                dict(diversity_weight=0.05, diversity_bandwidth=1e-300)])
def test_update_reduces_to_the_plain_update(kw):
    s = synth.subset(synth.c1(), 120)
    outs = []
    for extra in ({}, kw):
        cfg = oracle.make_config(voxel_resolution=s.r, loop_recency_gap=s.gap, **extra)
        pose, kp, L = s.pose12.copy(), s.kf_pose12.copy(), np.zeros(s.N)
        o = oracle.update(cfg, oracle.Keyframes(s.keyframes, s.D, s.r), s.D_now, pose, kp, L,
                          s.scan_mean3, s.scan_cov6, s.U)
        outs.append((pose, kp, L, o))
    for a, b in zip(outs[0][:3], outs[1][:3]):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(outs[0][3]["weight"], outs[1][3]["weight"])


def test_update_moves_translations_by_eta_d():
    """The whole update with eta > 0 differs from the plain one only in the translations, by
    fp32(t + eta d) with d taken at the translations the update started from (R35)."""
    s = synth.subset(synth.c1(), 60)
    eta, h = 0.02, 0.05
    plain = oracle.make_config(voxel_resolution=s.r, loop_recency_gap=s.gap,
                               posterior_floor=0.0, loglik_rel_floor=-np.inf)
    div = oracle.make_config(voxel_resolution=s.r, loop_recency_gap=s.gap, posterior_floor=0.0,
                             loglik_rel_floor=-np.inf, diversity_weight=eta,
                             diversity_bandwidth=h)
    kfs = oracle.Keyframes(s.keyframes, s.D, s.r)
    p0, k0 = s.pose12.copy(), s.kf_pose12.copy()
    oracle.update(plain, kfs, s.D_now, p0, k0, np.zeros(s.N), s.scan_mean3, s.scan_cov6, s.U)
    p1, k1 = s.pose12.copy(), s.kf_pose12.copy()
    oracle.update(div, kfs, s.D_now, p1, k1, np.zeros(s.N), s.scan_mean3, s.scan_cov6, s.U)
    t_start = s.pose12.reshape(-1, 3, 4)[:, :, 3].astype(np.float64)
    d = oracle.diversity(t_start, h)
    expect = (p0.reshape(-1, 3, 4)[:, :, 3].astype(np.float64) + eta * d).astype(np.float32)
    np.testing.assert_array_equal(p1.reshape(-1, 3, 4)[:, :, 3], expect)
    np.testing.assert_array_equal(p1.reshape(-1, 3, 4)[:, :, :3], p0.reshape(-1, 3, 4)[:, :, :3])
    np.testing.assert_array_equal(k1, k0)
    assert np.abs(eta * d).max() > 1e-4  # the term is not negligible in this case
