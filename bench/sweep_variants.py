"""Experiment harness: build libmcs variants (-D knobs) and time the C2 update phases of each.
    python bench/sweep_variants.py build   (here)    /  python bench/sweep_variants.py run (GPU)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANTS = {
    "tmem": [],
    "smem": ["MCS_SWEEP_TMEM_ACC=0"],
    "tmem_c896": ["MCS_SWEEP_CHUNK_PLANE=896"],
    "tmem_c672": ["MCS_SWEEP_CHUNK_PLANE=672"],
}
OUT = os.path.join(ROOT, "bench", "_variants")


def build():
    from paper_2504_18056_b200 import build as b
    for name, d in VARIANTS.items():
        b.build(defines=d, lib=os.path.join(OUT, f"libmcs_{name}.so"),
                build_dir=os.path.join(OUT, name))
        print("built", name)


def run_one(name):
    import numpy as np
    import paper_2504_18056_b200 as mcs
    import synth
    s = synth.c2()
    kw = dict(corr_mode=mcs.CORR_NN27, nn_radius=s.r) if name.startswith("nn27") else {}
    ctx = mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r, **kw)
    for (m3, c6), d in zip(s.keyframes, s.D):
        ctx.add_keyframe(m3, c6, d)
    ctx.set_particles(s.pose12, s.kf_pose12)
    ctx.snapshot()
    ctx.set_profiling(True)
    sw, sel, tot = [], [], []
    for k in range(8):
        ctx.restore()
        ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U, outputs=("loglik",))
        if k >= 3:
            ph = ctx.phase_ms()
            sw.append(ph["sweep"])
            sel.append(ph["select"])
            tot.append(ph["total"])
    print(json.dumps({"select_ms": float(np.median(sel)), "total_ms": float(np.median(tot))}),
          file=sys.stderr)
    return float(np.median(sw))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    elif sys.argv[1] == "one":
        print(json.dumps({"variant": sys.argv[2], "sweep_ms": run_one(sys.argv[2])}))
    else:
        for name in VARIANTS:
            env = dict(os.environ, MCS_LIB=os.path.join(OUT, f"libmcs_{name}.so"))
            r = subprocess.run([sys.executable, __file__, "one", name], env=env,
                               capture_output=True, text=True)
            print(r.stdout.strip(), r.stderr.strip()[-200:], flush=True)
