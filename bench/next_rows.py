"""Measurement of the NEXT rows and the flagged variants on the C2 workload, one
B200: prediction (Eq.1), keyframe-insertion overlap, keyframe registration (a0), the update
under NN27 correspondence, multi-iteration GN, post-update weighting and weight splitting, and
the per-frame driver at 100k particles.  Device time by CUDA events on the context stream
(updates: the library's phase events; single calls: events around the synchronous call, so
host work inside the call is included and said so).  L2 flushed before every timed call.

    python bench/next_rows.py > profiles/r01_next_rows.json        (on the GPU box)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2504_18056_b200 as mcs
    import synth
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 * 2**20, dtype=torch.float32, device=dev)
    s = synth.c2()
    N, S, K = s.N, s.S, s.K
    out = {"workload": "C2: 100k particles x 4096-pt scan vs 20 keyframes", "rows": {}}

    def ctx_for(**kw):
        c = mcs.Context(N, K + 1, S, loop_recency_gap=s.gap, voxel_resolution=s.r, **kw)
        for (m3, c6), d in zip(s.keyframes, s.D):
            c.add_keyframe(m3, c6, d)
        c.set_particles(s.pose12, s.kf_pose12)
        c.snapshot()
        return c

    def timed(fn, reps=5):
        ts = []
        for _ in range(reps + 2):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(1e3 * (time.perf_counter() - t0))
        return float(np.median(ts[2:]))

    # ---- update variants (library phase events)
    def update_ms(ctx, reps=5):
        ctx.set_profiling(True)
        tot, sw = [], []
        for k in range(reps + 2):
            ctx.restore()
            flush.fill_(1.0)
            torch.cuda.synchronize()
            ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, outputs=("loglik",))
            ph = ctx.phase_ms()
            if k >= 2:
                tot.append(ph["total"])
                sw.append(ph["sweep"])
        return float(np.median(tot)), float(np.median(sw))

    for name, kw in [("update_default", {}),
                     ("update_nn27", dict(corr_mode=mcs.CORR_NN27, nn_radius=s.r)),
                     ("update_gn_iterations_2", dict(gn_iterations=2)),
                     ("update_weight_after_update", dict(weight_after_update=1)),
                     ("update_clone_split", dict(clone_split=1)),
                     ("update_unmatched_penalty_1", dict(unmatched_penalty=1.0))]:
        with ctx_for(**kw) as c:
            t, sw = update_ms(c)
        out["rows"][name] = {"ms": t, "sweep_ms": sw, "evals_per_s": N * S / (t * 1e-3),
                             "config": kw and {k: float(v) for k, v in kw.items()}}
        print(name, t, file=sys.stderr, flush=True)

    with ctx_for() as c:
        # ---- prediction (Eq.1): one thread per particle, pose read + write (HBM)
        A = np.random.default_rng(0).normal(size=(6, 6)) * 0.02
        cov = A @ A.T + 1e-6 * np.eye(6)
        dT = synth.to12(synth.pose((0.0, 0.0, 0.01), (0.5, 0.0, 0.0)))
        t = timed(lambda: c.predict(dT, cov, 7, 3, vertical_sigma=0.1))
        out["rows"]["predict"] = {"ms_host_inclusive": t, "particles": N,
                                  "GBps_pose_rw": 2 * 48 * N / (t * 1e-3) / 1e9}
        # ---- overlap: the scan's pinned key path + one probe per point
        rel = synth.to12(np.linalg.inv(s.kf_gt[1]) @ s.T_gt)
        t = timed(lambda: c.overlap(s.scan_mean3, rel, 1), reps=20)
        out["rows"]["overlap"] = {"ms_host_inclusive": t, "scan_points": S,
                                  "rate": c.overlap(s.scan_mean3, rel, 1)}
        # ---- a0: registering one more keyframe (host cloud -> device table)
        m3, c6 = s.keyframes[0]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c.add_keyframe(m3, c6, s.D_now)
        torch.cuda.synchronize()
        out["rows"]["add_keyframe"] = {"ms_host_inclusive": 1e3 * (time.perf_counter() - t0),
                                       "points": int(len(m3))}

    # ---- the per-frame driver at 100k particles (prediction + update + overlap + insertion)
    tr = synth.corridor_lap(n_frames=14, S=S)
    init_cov = np.diag([0.05 ** 2] * 3 + [0.005 ** 2] * 3)
    frame_ms = []
    with mcs.MonteCarloSLAM(N, 32, S, init_pose=tr.gt[0], init_cov=init_cov, seed=3,
                            voxel_resolution=tr.r, loop_recency_gap=tr.gap) as g:
        for k in range(tr.F):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g.step(*tr.scans[k], tr.odom[k], tr.odom_cov, tr.D[k], U=int(tr.U[k]),
                   cloud=tr.clouds[k])
            torch.cuda.synchronize()
            frame_ms.append(1e3 * (time.perf_counter() - t0))
        K_end = g.K
    out["rows"]["driver_frame"] = {
        "ms_median_host_inclusive": float(np.median(frame_ms[2:])), "particles": N,
        "scan_points": S, "frames": tr.F, "keyframes_at_end": K_end,
        "frame_ms": [round(x, 3) for x in frame_ms],
        "note": "includes the read-back of every current pose, L and w each frame (6.4 MB); "
                "context: the paper reports ~50-60 ms per frame on an RTX 4090 (P:240)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
