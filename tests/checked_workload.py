"""Workloads run against the device-checked library build (MCS_LIB=libmcs_checked.so), by
tests/test_gpu_checked.py in a subprocess: every kernel family with its invariants checked on
device (index bounds, probe-loop termination, ladder / donor invariants).  Exits 0 when every
call succeeds and the results equal the plain build's (same kernels, checks only observe)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2504_18056_b200 as mcs  # noqa: E402
import synth  # noqa: E402


def ctx_for(s, N=None, **kw):
    N = s.N if N is None else N
    c = mcs.Context(N, max(s.K, 1), s.S, loop_recency_gap=s.gap, voxel_resolution=s.r, **kw)
    for (m3, c6), d in zip(s.keyframes, s.D):
        c.add_keyframe(m3, c6, d)
    c.set_particles(s.pose12[:N], s.kf_pose12[:N])
    return c


def main():
    out = {}
    s = synth.c1()
    for kw in ({}, dict(corr_mode=1, nn_radius=s.r), dict(clone_split=1, gn_iterations=2)):
        with ctx_for(s, **kw) as c:
            ev = c.eval(s.scan_mean3, s.scan_cov6)
            up = c.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
            st = c.get_particles()
        key = json.dumps(kw, sort_keys=True)
        out[key] = {"slot_n": int(ev["slot_n"].sum()), "n_dead": up["n_dead"],
                    "rep": up["representative"], "L": float(st["L"].sum()),
                    "pose": float(np.abs(st["pose12"]).sum())}
    # resampling with many dead and a ragged scan
    g = np.random.default_rng(1)
    with ctx_for(s) as c:
        e = g.random(s.N)
        dead = (g.random(s.N) < 0.6).astype(np.uint8)
        out["donor"] = int(c.resample(e, dead, 12345).sum())
        up = c.update(s.scan_mean3[:333], s.scan_cov6[:333], s.D_now, s.U)
        out["ragged"] = up["n_dead"]
    # multi-rank exchange path (in-process transport, 3 ranks on one device), migration-heavy
    G = 3
    tr = mcs.InprocTransport(G)
    import threading
    res = [None] * G
    parts = np.array_split(np.arange(s.N), G)

    errors = []

    def run(r):
        try:
            c = mcs.Context(len(parts[r]), s.K, s.S, loop_recency_gap=s.gap,
                            voxel_resolution=s.r, world_size=G, rank=r, transport=tr)
            for (m3, c6), d in zip(s.keyframes, s.D):
                c.add_keyframe(m3, c6, d)
            c.set_particles(s.pose12[parts[r]], s.kf_pose12[parts[r]])
            res[r] = c.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
            c.close()
        except Exception as e:
            errors.append(repr(e))

    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(G)]
    [t.start() for t in th]
    [t.join(300) for t in th]
    if errors or any(t.is_alive() for t in th):
        print("multirank failed:", errors, flush=True)
        os._exit(1)
    out["multirank_dead"] = int(sum(r["n_dead"] for r in res))
    # C2 subset: coherence sort, 20 keyframes, probe chains, propagation
    s2 = synth.subset(synth.c2(N=4000), 4000)
    with ctx_for(s2) as c:
        up = c.update(s2.scan_mean3, s2.scan_cov6, s2.D_now, s2.U)
        c.predict(synth.to12(np.eye(4)), np.eye(6) * 1e-4, 1, 1, vertical_sigma=0.1)
        ov = c.overlap(s2.scan_mean3, synth.to12(np.eye(4)), 0)
    out["c2"] = {"n_dead": up["n_dead"], "rep": up["representative"], "overlap": ov}
    print(json.dumps(out, sort_keys=True))


if __name__ == "__main__":
    main()
