"""Experiment: C2 sweep time vs the order of the scan points (random as generated, or sorted
along a space-filling curve).  The result of the update does not depend on the order beyond fp32
rounding of the per-stage sums."""
import json
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def morton3(p, cell):
    q = np.floor((p - p.min(0)) / cell).astype(np.int64)
    q = np.clip(q, 0, 1023)
    key = np.zeros(len(p), np.int64)
    for b in range(10):
        for a in range(3):
            key |= ((q[:, a] >> b) & 1) << (3 * b + a)
    return key


def main():
    import paper_2504_18056_b200 as mcs
    import synth
    s = synth.c2()
    orders = {"random (as generated)": np.arange(s.S)}
    for cell in (0.25, 0.5, 1.0, 2.0):
        orders[f"morton {cell} m"] = np.argsort(morton3(s.scan_mean3.astype(np.float64), cell),
                                                kind="stable")
    az = np.arctan2(s.scan_mean3[:, 1], s.scan_mean3[:, 0])
    orders["azimuth"] = np.argsort(az, kind="stable")
    c = mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r)
    for (m3, c6), d in zip(s.keyframes, s.D):
        c.add_keyframe(m3, c6, d)
    c.set_particles(s.pose12, s.kf_pose12)
    c.snapshot()
    c.set_profiling(True)
    for name, o in orders.items():
        m3 = np.ascontiguousarray(s.scan_mean3[o])
        c6 = np.ascontiguousarray(s.scan_cov6[o])
        sw = []
        for k in range(6):
            c.restore()
            c.update(m3, c6, s.D_now, s.U, outputs=())
            if k >= 2:
                sw.append(c.phase_ms()["sweep"])
        print(json.dumps({"order": name, "sweep_ms": float(np.median(sw))}), flush=True)


if __name__ == "__main__":
    main()
