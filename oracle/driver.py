"""Oracle twin of the per-frame loop (TEST INFRASTRUCTURE, NOT PRODUCT CODE).

The paper's three steps in its order, composed from the oracle's functions only:
prediction (Eq.1; elevator walk P:235), correction (orc_update: steps 2-11 of SURVEY
§8(c)), keyframe-list update by the voxel overlap with the last keyframe under the odometry's
relative motion (new keyframe pose of every particle := its current pose, R24),
representative.  Written independently of paper_2504_18056_b200/slam.py; only tests/
may use it.
"""
from __future__ import annotations

import numpy as np

from . import Keyframes, make_config, overlap, predict, update


def _pose12(T):
    return np.ascontiguousarray(np.asarray(T, np.float64)[:3, :4].reshape(12), np.float32)


class OracleSLAM:
    def __init__(self, N, init_pose, *, r, gap, init_cov=None, seed=0, overlap_threshold=0.7,
                 elevator_median_range=None, vertical_sigma=0.0, **cfg_kw):
        self.cfg = make_config(voxel_resolution=r, loop_recency_gap=gap, **cfg_kw)
        self.r = r
        self.N = N
        self.seed = int(seed)
        self.thr = overlap_threshold
        self.elev = elevator_median_range
        self.vs = vertical_sigma
        self.pose12 = np.tile(_pose12(init_pose), (N, 1))
        if init_cov is not None:
            predict(self.pose12, _pose12(np.eye(4)), np.asarray(init_cov, np.float64), self.seed,
                    0)
        self.kf_pose12 = np.zeros((N, 0, 12), np.float32)
        self.L = np.zeros(N)
        self.kfs = None
        self.kf_odom = None
        self.prev_odom = None
        self.frame = 0

    def step(self, scan_mean3, scan_cov6, odom_pose, odom_cov, D_t, U, cloud=None):
        cm, cc = (scan_mean3, scan_cov6) if cloud is None else cloud
        self.frame += 1
        odom_pose = np.asarray(odom_pose, np.float64)
        res = {"inserted": False, "overlap": None, "update": None, "elevator": False}
        if self.prev_odom is not None:  # prediction
            dT = np.linalg.solve(self.prev_odom, odom_pose)
            med = np.median(np.linalg.norm(np.asarray(scan_mean3, np.float64), axis=1))
            res["elevator"] = self.elev is not None and med < self.elev
            predict(self.pose12, _pose12(dT), np.asarray(odom_cov, np.float64), self.seed,
                    self.frame, 0, self.vs if res["elevator"] else 0.0)
        self.prev_odom = odom_pose
        if self.kfs is not None:  # correction
            res["update"] = update(self.cfg, self.kfs, float(D_t), self.pose12, self.kf_pose12,
                                   self.L, scan_mean3, scan_cov6, int(U))
        if self.kfs is None:  # keyframe list
            ins = True
        else:
            rel = np.linalg.solve(self.kf_odom, odom_pose)
            res["overlap"] = overlap(self.kfs.maps[-1], cm, _pose12(rel))
            ins = res["overlap"] < self.thr
        if ins:
            if self.kfs is None:
                self.kfs = Keyframes([(cm, cc)], np.array([float(D_t)]), self.r)
            else:
                self.kfs.append(cm, cc, float(D_t), self.r)
            self.kf_pose12 = np.ascontiguousarray(
                np.concatenate([self.kf_pose12, self.pose12[:, None, :]], axis=1))
            self.kf_odom = odom_pose
            res["inserted"] = True
        res["representative"] = res["update"]["representative"] if res["update"] else 0
        return res
