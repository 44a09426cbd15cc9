"""Debug: does one eval/update on a small context corrupt the host heap? (then stress imports)"""
import sys, os, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2504_18056_b200 as mcs
import synth

mode = sys.argv[1]
kw = dict(point_splits=int(sys.argv[2])) if len(sys.argv) > 2 else {}
s = synth.c1()
m3, c6 = s.keyframes[0]
if mode == "onept":
    kfs = [(m3[i:i + 1].copy(), c6[i:i + 1].copy()) for i in (0, 100, 900)]
    kp = np.ascontiguousarray(np.repeat(s.kf_pose12[:300], 3, axis=1))
    s = dataclasses.replace(s, keyframes=kfs, D=np.array([0.0, 1.0, 2.0]),
                            pose12=np.ascontiguousarray(s.pose12[:300]), kf_pose12=kp)
with mcs.Context(s.N, s.K, s.S, loop_recency_gap=s.gap, voxel_resolution=s.r, **kw) as ctx:
    for (a, b), d in zip(s.keyframes, s.D):
        ctx.add_keyframe(a, b, d)
    ctx.set_particles(s.pose12, s.kf_pose12)
    g = ctx.eval(s.scan_mean3, s.scan_cov6)
    print("eval ok", g["slot_n"].sum(), flush=True)
    if mode == "update":
        u = ctx.update(s.scan_mean3, s.scan_cov6, s.D_now, s.U)
        print("update ok", u["n_dead"], flush=True)
import compileall, importlib
for name in ["json", "email.mime.text", "http.server", "xml.dom.minidom", "unittest", "asyncio",
             "sqlite3", "csv", "decimal", "fractions", "statistics", "hypothesis"]:
    importlib.import_module(name)
print("imports ok", flush=True)
