"""C4 (1M particles x 8,192-point scan, 20 keyframes) on ONE B200: the per-GPU work of the
2/4/8-GPU configuration times G.  Library phase events, L2 flushed before each update."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2504_18056_b200 as mcs
    import synth
    s = synth.c4()
    flush = torch.empty(64 * 2**20, dtype=torch.float32, device="cuda")
    with mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r) as c:
        for (m3, c6), d in zip(s.keyframes, s.D):
            c.add_keyframe(m3, c6, d)
        c.set_particles(s.pose12, s.kf_pose12)
        c.snapshot()
        c.set_profiling(True)
        ph = []
        for k in range(5):
            c.restore()
            flush.fill_(1.0)
            torch.cuda.synchronize()
            c.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, outputs=())
            if k >= 2:
                ph.append(c.phase_ms())
    med = {k: float(np.median([p[k] for p in ph])) for k in ph[0]}
    print(json.dumps({"workload": "C4 on one GPU: 1M particles x 8192-pt scan, 20 keyframes",
                      "phase_ms": med,
                      "evals_per_s": s.N * s.S / (med["total"] * 1e-3)}))


if __name__ == "__main__":
    main()
