"""GPU parity of the boundary driven from plain C (examples/c_api_demo.c: one keyframe, 1,000
particles around the true pose, one mcs_update with host buffers) against the oracle on the
inputs the C program wrote out: l to 1e-4 relative, loop / updated / singular / clamped flags
exact, survivors' poses after the Gauss-Newton step to 1e-5 rad / 1e-5 m, and the respawn
(dead set, donors, representative) bit-exact from the GPU's l."""
import json
import subprocess

import numpy as np
import pytest

import oracle
from c_api_build import build_demo
from test_gpu_parity import L_RTOL, ROT_TOL, T_TOL, pose_err

pytestmark = pytest.mark.gpu


def _read(path):
    b = open(path, "rb").read()
    off = 0

    def take(dt, n):
        nonlocal off
        a = np.frombuffer(b, dtype=dt, count=n, offset=off)
        off += a.nbytes
        return a.copy()

    N, S = take(np.int32, 2)
    d = {"N": int(N), "S": int(S)}
    d["mean3"] = take(np.float32, 3 * S).reshape(S, 3)
    d["cov6"] = take(np.float32, 6 * S).reshape(S, 6)
    d["pose_in"] = take(np.float32, 12 * N).reshape(N, 12)
    d["D_now"] = float(take(np.float64, 1)[0])
    d["U"] = int(take(np.uint32, 1)[0])
    d["loglik"] = take(np.float64, N)
    d["psi6"] = take(np.float32, 6 * N).reshape(N, 6)
    d["weight"] = take(np.float64, N)
    d["donor"] = take(np.int32, N)
    d["flags"] = take(np.uint8, N)
    d["rep"] = int(take(np.int32, 1)[0])
    d["n_dead"] = int(take(np.int64, 1)[0])
    d["pose_out"] = take(np.float32, 12 * N).reshape(N, 12)
    assert off == len(b)
    return d


def test_c_program_update_matches_oracle(tmp_path):
    exe = build_demo(str(tmp_path))
    out = str(tmp_path / "io.bin")
    r = subprocess.run([exe, "1000", "512", out], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout, r.stderr)
    summary = json.loads(r.stdout.strip().splitlines()[-1])
    g = _read(out)
    N = g["N"]
    assert summary["N"] == N and summary["updated"] > 0
    kp = np.tile(np.eye(3, 4, dtype=np.float32).reshape(12), (N, 1))
    kfs = oracle.Keyframes([(g["mean3"], g["cov6"])], np.zeros(1), 0.5)
    cfg = oracle.make_config(voxel_resolution=0.5, loop_recency_gap=0)
    pose = g["pose_in"].copy()
    o = oracle.particles(cfg, kfs, g["D_now"], pose, kp.copy(), g["mean3"], g["cov6"])
    assert np.all(np.abs(g["loglik"] - o["loglik"]) <= L_RTOL * np.abs(o["loglik"]))
    np.testing.assert_array_equal(g["flags"] & 0x17, o["flags"] & 0x17)
    assert np.all(o["flags"] & 2)  # every particle loops and takes the GN step
    # respawn from the GPU's l (bit-exact contract, R17 / R18)
    L, e, w, _, _ = oracle.weights(np.zeros(N), g["loglik"])
    dead, nd = oracle.dead(g["loglik"], w)
    donor = oracle.resample(e, dead, g["U"])
    assert g["n_dead"] == nd
    np.testing.assert_array_equal(g["donor"], donor)
    L2 = L.copy()
    L2[donor >= 0] = L[donor[donor >= 0]]
    _, _, w2, _, _ = oracle.weights(L2)
    np.testing.assert_allclose(g["weight"], w2, rtol=1e-12, atol=1e-300)
    assert g["rep"] == oracle.representative(w2)
    # survivors keep their own updated pose; clones carry their donor's
    keep = donor < 0
    ang, dt = pose_err(g["pose_out"][keep], pose[keep])
    assert ang.max() <= ROT_TOL and dt.max() <= T_TOL, (ang.max(), dt.max())
    for i in np.nonzero(~keep)[0]:
        assert np.array_equal(g["pose_out"][i], g["pose_out"][donor[i]])
    # and the step moves the survivors towards the true pose (the identity)
    assert summary["survivor_t_err_out"] < summary["survivor_t_err_in"]
