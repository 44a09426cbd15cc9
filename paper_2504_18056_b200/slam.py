"""Per-frame driver of the method: the paper's three steps in its order around the
library's update.

    prediction      T_t^i = T_{t-1}^i dT_t exp(delta_t^i)           (Eq.1)
                    + the elevator heuristic's vertical random walk  (R32)
    correction      one `mcs_update`: neighbours, GICP likelihood + gradient, GN pose update,
                    keyframe propagation, weights, dead-particle pruning / respawn  (a1-a7)
    keyframe list   overlap of the scan with the last keyframe under the odometry's relative
                    motion; below the threshold (70 %) the scan becomes a keyframe and every
                    particle's new keyframe pose is its current pose (R24)
    representative  the largest-weight particle

Host logic only: every step of the path runs in libmcs kernels through the C-ABI (mcs.py).
The oracle's twin of this loop, written independently, is `oracle/driver.py`.
"""
from __future__ import annotations

import numpy as np

from .mcs import Context


def _to12(T) -> np.ndarray:
    T = np.asarray(T, np.float64)
    return np.ascontiguousarray(T[:3, :4].reshape(12), dtype=np.float32)


def _to44(p12) -> np.ndarray:
    T = np.eye(4)
    T[:3, :4] = np.asarray(p12, np.float64).reshape(3, 4)
    return T


def in_elevator(scan_mean3, median_range: float | None) -> bool:
    """'a simple heuristic ... based on the threshold of the median of point distances'
    (R32): the sensor is in the elevator when the median range of the scan is below the
    threshold (the cabin walls are close in every direction)."""
    if median_range is None:
        return False
    return float(np.median(np.linalg.norm(np.asarray(scan_mean3, np.float64), axis=1))) \
        < median_range


class MonteCarloSLAM:
    """Gradient-guided Monte Carlo SLAM on one GPU (or one particle shard of a multi-GPU job,
    when `world_size`, `rank` and `nccl_unique_id` are passed through to the Context)."""

    def __init__(self, n_particles: int, capacity_keyframes: int, capacity_scan_points: int, *,
                 init_pose, init_cov=None, seed: int = 0, overlap_threshold: float = 0.7,
                 elevator_median_range: float | None = None, vertical_sigma: float = 0.0,
                 outputs=("donor",), **cfg):
        self.ctx = Context(n_particles, capacity_keyframes, capacity_scan_points, **cfg)
        self.N = n_particles
        self.seed = int(seed)
        self.overlap_threshold = float(overlap_threshold)
        self.elevator_median_range = elevator_median_range
        self.vertical_sigma = float(vertical_sigma)
        self.outputs = tuple(outputs)  # per-particle update outputs read back each frame
        self.frame = 0
        self.K = 0
        self.prev_odom = None
        self.kf_odom = None
        self.ctx.set_particles(np.tile(_to12(init_pose), (n_particles, 1)))
        if init_cov is not None:  # initial spread: Eq.1 with dT = I (frame 0 of the stream)
            self.ctx.predict(_to12(np.eye(4)), np.asarray(init_cov, np.float64), self.seed, 0)
        self._rng = np.random.default_rng(self.seed)

    def close(self):
        self.ctx.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def step(self, scan_mean3, scan_cov6, odom_pose, odom_cov, path_length: float,
             U: int | None = None, cloud=None, state: bool = False) -> dict:
        """One frame.  scan (S,3)/(S,6) fp32 in the sensor frame (the correction's points);
        cloud = (mean3, cov6) the whole frame downsampled at r, used for the overlap test and
        registered as the keyframe (default: the scan); odom_pose the odometry pose T^o_t
        (4x4); odom_cov the (6,6) covariance of the relative motion (rho, phi); path_length the
        cumulative odometry path length D_t (R14); U the resampling uniform (uint32; drawn from
        the seeded generator when None); state: also return every particle's pose, L and weight
        (and keyframe poses) in out["state"]."""
        cloud_m, cloud_c = (scan_mean3, scan_cov6) if cloud is None else cloud
        self.frame += 1
        odom_pose = np.asarray(odom_pose, np.float64)
        U = int(self._rng.integers(0, 2**32)) if U is None else int(U)
        out = {"frame": self.frame, "inserted": False, "overlap": None, "update": None,
               "elevator": False}
        # (1) prediction (Eq.1)
        if self.prev_odom is not None:
            dT = np.linalg.inv(self.prev_odom) @ odom_pose
            out["elevator"] = in_elevator(scan_mean3, self.elevator_median_range)
            self.ctx.predict(_to12(dT), np.asarray(odom_cov, np.float64), self.seed, self.frame,
                             vertical_sigma=self.vertical_sigma if out["elevator"] else 0.0)
        self.prev_odom = odom_pose
        # (2) correction (needs a keyframe)
        if self.K > 0:
            out["update"] = self.ctx.update(scan_mean3, scan_cov6, float(path_length), U,
                                            outputs=self.outputs)
        # (3) keyframe list
        if self.K == 0:
            insert = True
        else:
            rel = np.linalg.inv(self.kf_odom) @ odom_pose
            out["overlap"] = self.ctx.overlap(cloud_m, _to12(rel), self.K - 1)
            insert = out["overlap"] < self.overlap_threshold
        if insert:
            self.ctx.add_keyframe(cloud_m, cloud_c, float(path_length))
            self.kf_odom = odom_pose
            self.K += 1
            out["inserted"] = True
        # (4) representative
        # the representative is a GLOBAL index: its owner's pose reaches every rank (collective)
        rep = out["update"]["representative"] if out["update"] is not None else 0
        out["representative"] = int(rep)
        out["pose"] = _to44(self.ctx.get_global_pose(rep))
        if state:
            out["state"] = self.ctx.get_particles()
        return out
