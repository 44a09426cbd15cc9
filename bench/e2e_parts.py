"""Where the end-to-end (synchronous mcs_update, pinned host buffers) time goes beyond the
device-timed update: no outputs vs loglik + weight, against the profiled device total."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2504_18056_b200 as mcs  # noqa: E402
import synth  # noqa: E402

s = synth.c2()
ctx = mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r)
for (m3, c6), d in zip(s.keyframes, s.D):
    ctx.add_keyframe(m3, c6, d)
ctx.set_particles(s.pose12, s.kf_pose12)
ctx.snapshot()
h_m = torch.from_numpy(s.scan_mean3).pin_memory()
h_c = torch.from_numpy(s.scan_cov6).pin_memory()
h_out = {"loglik": torch.empty(s.N, dtype=torch.float64).pin_memory(),
         "weight": torch.empty(s.N, dtype=torch.float64).pin_memory()}
for name, out in (("no outputs", None), ("loglik + weight", h_out), ("no outputs", None),
                  ("loglik + weight", h_out)):
    ts = []
    for k in range(25):
        ctx.restore()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ctx.update(h_m, h_c, s.D_now, s.U, outputs=(), out=out)
        t2 = time.perf_counter()
        if k >= 5:
            ts.append(t2 - t1)
    print(name, round(1e3 * float(np.median(ts)), 4), "ms")
ctx.set_profiling(True)
ph = []
for k in range(10):
    ctx.restore()
    ctx.update(h_m, h_c, s.D_now, s.U, outputs=(), out=None)
    if k >= 3:
        ph.append(ctx.phase_ms()["total"])
print("device (phase total)", round(float(np.median(ph)), 4), "ms")
