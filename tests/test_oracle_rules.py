"""Pins for oracle rules that no other pin reaches (round-1 verdict, "What's weak" 1):

* R4, the G-slot combine (Fig.3 caption P:108): with one old and one recent neighbour,
  H and b come from the old slot alone while l sums both (Eq.2);
* R8, the unmatched penalty: l = sum_s l_s - kappa * #unmatched (point, slot) pairs;
* P:190's posterior floor: a particle whose normalised posterior is below 1e-8 dies even when
  its log-likelihood equals the best one;
* R13, the weighting likelihood: pre-update (default) or re-evaluated after the GN step (flag).

Every expected value is hand algebra recorded in tests/golden/hand_cases.json with its citation;
none is produced by the oracle or by the CUDA path.  CPU only.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_cases.json")))


def _pose12(t):
    T = np.zeros((3, 4), np.float32)
    T[:, :3] = np.eye(3, dtype=np.float32)
    T[:, 3] = t
    return T.reshape(12)


def _two_slot(gn_slots=0, kappa=0.0, with_unmatched=False):
    h = GOLD["two_slot_old_recent"]
    cloud = (np.array([h["mu_prime"]], np.float32), np.array([h["cov6_prime"]], np.float32))
    kfs = oracle.Keyframes([cloud, cloud], [0.0, 1.0], h["r"])
    cfg = oracle.make_config(voxel_resolution=h["r"], neighbor_count=h["neighbor_count"],
                             loop_recency_gap=h["loop_recency_gap"], gn_slots=gn_slots,
                             unmatched_penalty=kappa)
    mu = [h["mu"]] + ([h["unmatched_point"]] if with_unmatched else [])
    cov = [h["cov6"]] * len(mu)
    pose = _pose12(h["pose_t"])[None].copy()
    kp = np.stack([_pose12(t) for t in h["kf_t"]])[None].copy()
    out = oracle.particles(cfg, kfs, 2.0, pose, kp, np.array(mu, np.float32),
                           np.array(cov, np.float32), apply_update=False, slots=True)
    return h, out


def test_r4_old_slot_alone_drives_the_update():
    h, out = _two_slot()
    assert list(out["slot_kf"][0]) == [0, 1] and out["flags"][0] & 1  # loop via the old slot
    np.testing.assert_array_equal(out["slot_l"][0], h["l_per_slot"])
    assert out["loglik"][0] == h["loglik"]  # l over every neighbour (Eq.2)
    np.testing.assert_array_equal(out["grad6"][0], h["grad6_old_slots"])
    np.testing.assert_array_equal(out["hess36"][0], np.diag(h["H_diag_old_slots"]))


def test_r4_all_slots_flag_sums_both():
    h, out = _two_slot(gn_slots=1)
    assert out["loglik"][0] == h["loglik"]
    np.testing.assert_array_equal(out["grad6"][0], h["grad6_all_slots"])
    np.testing.assert_array_equal(out["hess36"][0], np.diag(h["H_diag_all_slots"]))


def test_r4_no_old_slot_gives_zero_gradient_and_no_loop():
    """gap larger than the keyframe count: no neighbour is old => no loop, G empty, g = 0."""
    h = GOLD["two_slot_old_recent"]
    cloud = (np.array([h["mu_prime"]], np.float32), np.array([h["cov6_prime"]], np.float32))
    kfs = oracle.Keyframes([cloud, cloud], [0.0, 1.0], h["r"])
    cfg = oracle.make_config(voxel_resolution=h["r"], neighbor_count=2, loop_recency_gap=2)
    pose = _pose12(h["pose_t"])[None].copy()
    kp = np.stack([_pose12(t) for t in h["kf_t"]])[None].copy()
    out = oracle.particles(cfg, kfs, 2.0, pose, kp, np.array([h["mu"]], np.float32),
                           np.array([h["cov6"]], np.float32))
    assert out["flags"][0] == 0 and out["loglik"][0] == h["loglik"]
    assert not out["grad6"][0].any() and not out["hess36"][0].any() and not out["psi6"][0].any()


@pytest.mark.parametrize("gn_slots", [0, 1])
def test_r8_unmatched_penalty_closed_form(gn_slots):
    h, out0 = _two_slot(gn_slots=gn_slots, with_unmatched=True)
    assert list(out0["slot_n"][0]) == [1, 1]  # the far point is unmatched in both slots
    assert out0["loglik"][0] == h["loglik"]  # kappa = 0: skipped
    _, out = _two_slot(gn_slots=gn_slots, kappa=h["kappa"], with_unmatched=True)
    assert out["loglik"][0] == h["loglik_with_kappa"]
    np.testing.assert_array_equal(out["grad6"][0], out0["grad6"][0])  # kappa is not in g


@pytest.mark.parametrize("case", GOLD["posterior_floor"]["cases"])
def test_p190_posterior_floor_alone(case):
    h = GOLD["posterior_floor"]
    L, e, w, _, _ = oracle.weights(np.array(case["L_prev"]), np.array(h["l"]))
    np.testing.assert_allclose(w[1], case["w1"], rtol=1e-12)
    d, nd = oracle.dead(np.array(h["l"]), w)
    assert list(d) == case["dead"] and nd == sum(case["dead"])
    # the relative log-likelihood floor alone never kills an equal-l particle
    d2, _ = oracle.dead(np.array(h["l"]), w, post_floor=0.0)
    assert not d2.any()


@pytest.mark.parametrize("case", GOLD["posterior_floor"]["cases"])
def test_p190_posterior_floor_through_the_whole_update(case):
    """Two identical particles (equal l), prior log-weights L_prev: particle 1 is respawned from
    particle 0 exactly when its posterior is below 1e-8 (flags bit3, donor 0)."""
    g = GOLD["gicp_hand_case"]
    cloud = (np.array([g["mu_prime"]], np.float32), np.array([g["cov6_prime"]], np.float32))
    kfs = oracle.Keyframes([cloud], [0.0], g["r"])
    cfg = oracle.make_config(voxel_resolution=g["r"], loop_recency_gap=1)  # no loop: no update
    pose = np.stack([_pose12(g["rel_translation"])] * 2).copy()
    kp = np.stack([_pose12([0, 0, 0])] * 2)[:, None].copy()
    L = np.array(case["L_prev"], np.float64)
    out = oracle.update(cfg, kfs, 1.0, pose, kp, L, np.array([g["mu"]], np.float32),
                        np.array([g["cov6"]], np.float32), 12345)
    assert out["status"] == 0 and out["loglik"][0] == out["loglik"][1] == g["loglik"]
    assert [(f >> 3) & 1 for f in out["flags"]] == case["dead"]
    assert out["n_dead"] == sum(case["dead"])
    assert list(out["donor"]) == ([-1, 0] if case["dead"][1] else [-1, -1])


@pytest.mark.parametrize("post", [0, 1])
def test_r13_weighting_likelihood_pre_or_post_update(post):
    """R13 (Eq.11 after §III-C): the weighting l is the pre-update l of the sweep that
    linearised (default), or re-evaluated at the updated pose (flag).  Hand case (golden): one
    point, Omega = I, e = (-1, 0, 0) => pre-update l = -1; one damped GN step (lambda = 5e-7)
    leaves the fp32 translation t = fp32(1 - 1/(1 + 5e-7)) => post-update l = -t^2."""
    g = GOLD["gicp_hand_case"]
    cloud = (np.array([g["mu_prime"]], np.float32), np.array([g["cov6_prime"]], np.float32))
    kfs = oracle.Keyframes([cloud], [0.0], g["r"])
    cfg = oracle.make_config(voxel_resolution=g["r"], loop_recency_gap=0, posterior_floor=0.0,
                             loglik_rel_floor=-np.inf, weight_after_update=post)
    pose = _pose12(g["rel_translation"])[None].copy()
    kp = _pose12([0, 0, 0])[None, None].copy()
    out = oracle.update(cfg, kfs, 1.0, pose, kp, np.zeros(1), np.array([g["mu"]], np.float32),
                        np.array([g["cov6"]], np.float32), 7)
    t = np.float32(1.0 - 1.0 / (1.0 + 5e-7))
    assert pose[0, 3] == t
    expect = -(float(t) ** 2) if post else g["loglik"]
    np.testing.assert_allclose(out["loglik"][0], expect, rtol=1e-12)
