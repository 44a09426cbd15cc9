"""The per-frame loop (prediction -> correction -> keyframe list -> representative).

CPU: the oracle twin (oracle/driver.py) on a short corridor trajectory with exact odometry
tracks the ground truth, inserts keyframes by the 70 % overlap rule, and the
elevator heuristic (R32) only switches the vertical walk on.
GPU: the product driver (paper_2504_18056_b200/slam.py, every step in libmcs kernels) equals
the oracle twin frame by frame, and closes the loop of a drifting 160 m lap.
"""
import functools

import numpy as np
import pytest

import oracle
import synth
from oracle.driver import OracleSLAM


@functools.lru_cache(maxsize=4)
def _traj(n_frames, S, sig_t, sig_r, step=2.0):
    return synth.corridor_lap(n_frames=n_frames, S=S, sig_t=sig_t, sig_r=sig_r, step=step)


def _terr(T, G):
    return float(np.linalg.norm(np.asarray(T)[:3, 3] - G[:3, 3]))


def test_oracle_driver_tracks_ground_truth_with_exact_odometry():
    tr = _traj(10, 512, 0.0, 0.0)
    init_cov = np.diag([0.05 ** 2] * 3 + [0.005 ** 2] * 3)
    slam = OracleSLAM(48, tr.gt[0], r=tr.r, gap=tr.gap, init_cov=init_cov, seed=3)
    inserted = []
    for k in range(tr.F):
        res = slam.step(*tr.scans[k], tr.odom[k], np.zeros((6, 6)), tr.D[k], tr.U[k],
                        cloud=tr.clouds[k])
        inserted.append(res["inserted"])
        if res["overlap"] is not None:
            assert res["inserted"] == (res["overlap"] < 0.7)
        rep = slam.pose12[res["representative"]].reshape(3, 4)
        T = np.eye(4)
        T[:3] = rep
        assert _terr(T, tr.gt[k]) < 0.25, (k, _terr(T, tr.gt[k]))
    assert inserted[0] and 1 < sum(inserted) < tr.F
    assert slam.kf_pose12.shape[1] == sum(inserted)


def test_elevator_heuristic_switches_the_vertical_walk():
    from paper_2504_18056_b200.slam import in_elevator
    near = np.random.default_rng(0).normal(0, 0.5, (200, 3))
    far = near * 20
    assert in_elevator(near, 1.5) and not in_elevator(far, 1.5) and not in_elevator(near, None)
    # oracle twin: the walk moves only z and only when the heuristic fires
    tr = _traj(10, 512, 0.0, 0.0)
    a = OracleSLAM(16, tr.gt[0], r=tr.r, gap=tr.gap, seed=1, elevator_median_range=1e6,
                   vertical_sigma=0.5)
    b = OracleSLAM(16, tr.gt[0], r=tr.r, gap=tr.gap, seed=1)
    for s in (a, b):
        s.step(*tr.scans[0], tr.odom[0], np.zeros((6, 6)), tr.D[0], tr.U[0])
        s.prev_odom = tr.odom[0]
    pa, pb = a.pose12.copy(), b.pose12.copy()
    from oracle import predict
    predict(pa, synth.to12(np.eye(4)), np.zeros((6, 6)), 1, 2, 0, 0.5)
    d = pa.reshape(-1, 3, 4) - pb.reshape(-1, 3, 4)
    assert np.all(d[:, :, :3] == 0) and np.all(d[:, :2, 3] == 0) and np.abs(d[:, 2, 3]).max() > 0


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_driver_equals_oracle_twin_frame_by_frame():
    import paper_2504_18056_b200 as mcs
    tr = _traj(12, 512, 0.02, 0.002)
    N = 256
    init_cov = np.diag([0.1 ** 2] * 3 + [0.01 ** 2] * 3)
    o = OracleSLAM(N, tr.gt[0], r=tr.r, gap=tr.gap, init_cov=init_cov, seed=7)
    with mcs.MonteCarloSLAM(N, 16, 512, init_pose=tr.gt[0], init_cov=init_cov, seed=7,
                            voxel_resolution=tr.r, loop_recency_gap=tr.gap) as g:
        for k in range(tr.F):
            ro = o.step(*tr.scans[k], tr.odom[k], tr.odom_cov, tr.D[k], tr.U[k],
                        cloud=tr.clouds[k])
            rg = g.step(*tr.scans[k], tr.odom[k], tr.odom_cov, tr.D[k], U=int(tr.U[k]),
                        cloud=tr.clouds[k], state=True)
            assert rg["inserted"] == ro["inserted"], k
            if ro["overlap"] is not None:
                assert rg["overlap"] == ro["overlap"], k  # exact: pinned fp32 cells, both sides
            if ro["update"] is not None:
                assert rg["update"]["n_dead"] == ro["update"]["n_dead"], k
                np.testing.assert_array_equal(rg["update"]["donor"], ro["update"]["donor"])
                assert rg["representative"] == ro["representative"], k
            P = rg["state"]["pose12"].reshape(-1, 3, 4).astype(np.float64)
            Q = o.pose12.reshape(-1, 3, 4)
            assert np.abs(P - Q).max() < 1e-4, (k, np.abs(P - Q).max())


@pytest.mark.gpu
def test_driver_closes_the_loop_of_a_drifting_lap():
    import paper_2504_18056_b200 as mcs
    tr = _traj(88, 1024, 0.03, 0.003)
    N = 20000
    init_cov = np.diag([0.05 ** 2] * 3 + [0.005 ** 2] * 3)
    with mcs.MonteCarloSLAM(N, 96, 1024, init_pose=tr.gt[0], init_cov=init_cov, seed=11,
                            voxel_resolution=tr.r, loop_recency_gap=tr.gap) as g:
        errs = []
        for k in range(tr.F):
            rg = g.step(*tr.scans[k], tr.odom[k], tr.odom_cov, tr.D[k], U=int(tr.U[k]),
                        cloud=tr.clouds[k])
            errs.append(_terr(rg["pose"], tr.gt[k]))
        K = g.K
    odo = _terr(tr.odom[-1], tr.gt[-1])
    print(f"keyframes {K}, odometry error {odo:.2f} m, representative error {errs[-1]:.2f} m")
    assert odo > 0.8                    # the odometry drifted (1.10 m with these seeds)
    assert errs[-1] < 0.5 * odo and errs[-1] < 0.5


@pytest.mark.gpu
def test_two_rank_driver_equals_one_rank():
    """The driver on two particle shards (two contexts joined by the in-process transport, one
    host thread per rank): the representative is a GLOBAL index and every rank reads its pose
    through the collective mcs_get_global_pose; frame by frame it equals the one-rank driver."""
    import threading

    import paper_2504_18056_b200 as mcs
    tr = _traj(8, 512, 0.02, 0.002)
    N = 256
    init_cov = np.diag([0.1 ** 2] * 3 + [0.01 ** 2] * 3)

    def run(world, rank, n, transport, sink):
        kw = dict(voxel_resolution=tr.r, loop_recency_gap=tr.gap)
        if world > 1:
            kw.update(world_size=world, rank=rank, transport=transport)
        out = []
        with mcs.MonteCarloSLAM(n, 16, 512, init_pose=tr.gt[0], init_cov=init_cov, seed=7,
                                **kw) as g:
            for k in range(tr.F):
                r = g.step(*tr.scans[k], tr.odom[k], tr.odom_cov, tr.D[k], U=int(tr.U[k]),
                           cloud=tr.clouds[k])
                out.append((r["inserted"], r["representative"], r["pose"]))
        sink[rank] = out

    one = {}
    run(1, 0, N, None, one)
    tp = mcs.InprocTransport(2)
    two, errors = {}, []

    def worker(rank):
        try:
            run(2, rank, N // 2, tp, two)
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not errors, errors
    for k in range(tr.F):
        for rank in range(2):
            ins, rep, pose = two[rank][k]
            assert ins == one[0][k][0] and rep == one[0][k][1], (k, rank)
            np.testing.assert_array_equal(pose, one[0][k][2])
