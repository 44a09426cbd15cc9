"""CPU oracle for the MCS hot path — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  It wraps the plain C
oracle ``mcs_oracle.c`` (fp64, written step by step from the paper; see its
header for citations) through ctypes.  It shares no code with
``paper_2504_18056_b200`` and never imports it.

Parity unpinned: absolute likelihood scale on synthetic scenes, the pruning
threshold semantics (R17), pre- vs post-update weighting (R13), and
Eq.10's frame convention (R16) — nothing outside the oracle fixes them.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mcs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

LN_1E16 = float(np.log(1e-16))


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no contraction: the fp32 key path is pinned, R27)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "mcs_oracle.h"))
    ):
        cmd = ["gcc", "-std=gnu11", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class Config(C.Structure):
    _fields_ = [
        ("neighbor_count", C.c_int32),
        ("loop_recency_gap", C.c_int32),
        ("voxel_resolution", C.c_float),
        ("gn_slots", C.c_int32),
        ("damping_rel", C.c_double),
        ("step_clamp", C.c_double),
        ("unmatched_penalty", C.c_double),
        ("loglik_rel_floor", C.c_double),
        ("posterior_floor", C.c_double),
        ("gn_iterations", C.c_int32),
        ("weight_after_update", C.c_int32),
        ("corr_mode", C.c_int32),
        ("nn_radius", C.c_float),
        ("clone_split", C.c_int32),
        ("diversity_weight", C.c_double),
        ("diversity_bandwidth", C.c_double),
    ]


CORR_CELL, CORR_NN27 = 0, 1


def make_config(voxel_resolution=0.5, neighbor_count=3, loop_recency_gap=10, gn_slots=0,
                damping_rel=1e-6, step_clamp=1.0, unmatched_penalty=0.0,
                loglik_rel_floor=LN_1E16, posterior_floor=1e-8, gn_iterations=1,
                weight_after_update=0, corr_mode=CORR_CELL, nn_radius=0.0,
                clone_split=0, diversity_weight=0.0, diversity_bandwidth=1.0) -> Config:
    return Config(neighbor_count, loop_recency_gap, voxel_resolution, gn_slots, damping_rel,
                  step_clamp, unmatched_penalty, loglik_rel_floor, posterior_floor,
                  gn_iterations, weight_after_update, corr_mode, nn_radius, clone_split,
                  diversity_weight, diversity_bandwidth)


class ParticleOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "loglik", "grad6", "hess36", "psi6", "flags",
        "slot_l", "slot_H36", "slot_b6", "slot_n", "slot_kf")]


class UpdateOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "loglik", "grad6", "hess36", "psi6", "weight", "donor", "flags",
        "representative", "n_dead")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        vp, i32, f32, f64, u32 = C.c_void_p, C.c_int32, C.c_float, C.c_double, C.c_uint32
        L.orc_se3_exp.argtypes = [vp, vp]
        L.orc_se3_log.argtypes = [vp, vp]
        L.orc_se3_log.restype = C.c_int
        L.orc_compose.argtypes = [vp, vp, vp]
        L.orc_map_build.argtypes = [vp, vp, i32, f32]
        L.orc_map_build.restype = vp
        L.orc_map_free.argtypes = [vp]
        L.orc_map_size.argtypes = [vp]
        L.orc_map_size.restype = i32
        L.orc_map_lookup.argtypes = [vp, i32, i32, i32, vp, vp]
        L.orc_map_lookup.restype = i32
        L.orc_map_cell.argtypes = [vp, i32, vp, vp]
        L.orc_map_cell.restype = i32
        L.orc_map_set_corr.argtypes = [vp, i32, f32]
        L.orc_map_correspond.argtypes = [vp, vp]
        L.orc_map_correspond.restype = i32
        L.orc_cell_of.argtypes = [f32, f32, f32, f32, vp]
        L.orc_cell_of.restype = C.c_int
        L.orc_relpose.argtypes = [vp, vp, vp, vp]
        L.orc_pair_linearize.argtypes = [vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp]
        L.orc_pair_linearize.restype = C.c_int
        L.orc_pair_loglik_frozen.argtypes = [vp, vp, i32, vp, vp, vp]
        L.orc_pair_loglik_frozen.restype = f64
        L.orc_pair_omegas.argtypes = [vp, vp, i32, vp, vp, vp]
        L.orc_gn_step.argtypes = [vp, vp, f64, f64, vp, vp]
        L.orc_gn_step.restype = C.c_int
        L.orc_propagation_ratio.argtypes = [vp, i32, i32, f64, vp]
        L.orc_propagation_ratio.restype = C.c_int
        L.orc_particles.argtypes = [vp, i32, vp, vp, f64, i32, vp, vp, i32, vp, vp, i32, vp,
                                    i32, i32, vp]
        L.orc_particles.restype = C.c_int
        L.orc_weights.argtypes = [i32, vp, vp, vp, vp, vp, vp]
        L.orc_dead.argtypes = [i32, vp, vp, f64, f64, vp]
        L.orc_dead.restype = C.c_int64
        L.orc_resample.argtypes = [i32, vp, vp, u32, vp]
        L.orc_resample.restype = C.c_int
        L.orc_diversity.argtypes = [i32, vp, f64, vp]
        L.orc_representative.argtypes = [i32, vp]
        L.orc_representative.restype = i32
        L.orc_update.argtypes = [vp, i32, vp, vp, f64, i32, vp, vp, i32, vp, vp, vp, i32, u32, vp]
        L.orc_update.restype = C.c_int
        L.orc_num_threads.restype = C.c_int
        L.orc_set_num_threads.argtypes = [C.c_int]
        L.orc_philox4x32_10.argtypes = [vp, vp, vp]
        L.orc_normals8.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, vp]
        L.orc_predict.argtypes = [i32, vp, vp, vp, C.c_uint64, C.c_uint64, C.c_int64, f64]
        L.orc_predict.restype = C.c_int
        L.orc_overlap.argtypes = [vp, vp, i32, vp]
        L.orc_overlap.restype = f64
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


# ---------------------------------------------------------------- SE(3)
def se3_exp(xi) -> np.ndarray:
    xi = _c(xi, np.float64)
    T = np.zeros(12, np.float64)
    lib().orc_se3_exp(_p(xi), _p(T))
    return T.reshape(3, 4)


def se3_log(T) -> np.ndarray:
    T = _c(np.asarray(T, np.float64).reshape(12), np.float64)
    xi = np.zeros(6, np.float64)
    if lib().orc_se3_log(_p(T), _p(xi)):
        raise ValueError("rotation angle at pi: log ill-conditioned")
    return xi


def compose(A, B) -> np.ndarray:
    A = _c(np.asarray(A).reshape(12), np.float64)
    B = _c(np.asarray(B).reshape(12), np.float64)
    out = np.zeros(12, np.float64)
    lib().orc_compose(_p(A), _p(B), _p(out))
    return out.reshape(3, 4)


# ---------------------------------------------------------------- voxel map
class Map:
    """Keyframe voxel map: one aggregate per occupied fp32 cell."""

    def __init__(self, mean3, cov6, r: float):
        self.mean3 = _c(mean3, np.float32).reshape(-1, 3)
        self.cov6 = _c(cov6, np.float32).reshape(-1, 6)
        self.r = float(r)
        self.ptr = lib().orc_map_build(_p(self.mean3), _p(self.cov6), len(self.mean3), self.r)

    def __len__(self):
        return int(lib().orc_map_size(self.ptr))

    def lookup(self, cell):
        m = np.zeros(3, np.float64)
        c = np.zeros(6, np.float64)
        cnt = lib().orc_map_lookup(self.ptr, int(cell[0]), int(cell[1]), int(cell[2]), _p(m), _p(c))
        return (cnt, m, c) if cnt else (0, None, None)

    def set_corr(self, mode: int, nn_radius: float = 0.0):
        """Correspondence rule for pair_linearize / overlap-free queries: CELL (R7) or NN27 (R33)."""
        lib().orc_map_set_corr(self.ptr, int(mode), float(nn_radius))

    def correspond(self, q) -> int:
        """Sorted-list index of the cell matched by the fp32 point q under the map's rule, or -1."""
        q = _c(np.asarray(q, np.float32).reshape(3), np.float32)
        return int(lib().orc_map_correspond(self.ptr, _p(q)))

    def cells(self, idx):
        """(mean (n,3), cov6 (n,6)) fp64 of the cells at sorted-list indices idx."""
        idx = np.asarray(idx)
        mean = np.zeros((len(idx), 3))
        cov = np.zeros((len(idx), 6))
        for j, k in enumerate(idx):
            lib().orc_map_cell(self.ptr, int(k), mean[j].ctypes.data, cov[j].ctypes.data)
        return mean, cov

    def __del__(self):
        try:
            if self.ptr:
                lib().orc_map_free(self.ptr)
        except Exception:
            pass


def cell_of(q, r: float):
    c = np.zeros(3, np.int32)
    ok = lib().orc_cell_of(float(np.float32(q[0])), float(np.float32(q[1])),
                           float(np.float32(q[2])), float(np.float32(1.0) / np.float32(r)), _p(c))
    return c if ok else None


def relpose(Tk, Tt):
    Tk = _c(np.asarray(Tk).reshape(12), np.float32)
    Tt = _c(np.asarray(Tt).reshape(12), np.float32)
    r32 = np.zeros(12, np.float32)
    r64 = np.zeros(12, np.float64)
    lib().orc_relpose(_p(Tk), _p(Tt), _p(r32), _p(r64))
    return r32.reshape(3, 4), r64.reshape(3, 4)


@dataclass
class PairResult:
    l: float
    H: np.ndarray
    b: np.ndarray
    n: int
    corr: np.ndarray


def pair_linearize(m: Map, mean3, cov6, rel32, rel64) -> PairResult:
    mean3 = _c(mean3, np.float32).reshape(-1, 3)
    cov6 = _c(cov6, np.float32).reshape(-1, 6)
    rel32 = _c(np.asarray(rel32).reshape(12), np.float32)
    rel64 = _c(np.asarray(rel64).reshape(12), np.float64)
    S = len(mean3)
    l = C.c_double()
    n = C.c_int32()
    H = np.zeros(36, np.float64)
    b = np.zeros(6, np.float64)
    corr = np.zeros(S, np.int32)
    rc = lib().orc_pair_linearize(m.ptr, _p(mean3), _p(cov6), S, _p(rel32), _p(rel64),
                                  C.byref(l), _p(H), _p(b), C.byref(n), _p(corr))
    if rc:
        raise FloatingPointError("non-PD combined covariance")
    return PairResult(l.value, H.reshape(6, 6), b, n.value, corr)


def pair_omegas(m: Map, cov6, rel64, corr):
    cov6 = _c(cov6, np.float32).reshape(-1, 6)
    rel64 = _c(np.asarray(rel64).reshape(12), np.float64)
    corr = _c(corr, np.int32)
    om = np.zeros((len(cov6), 9), np.float64)
    lib().orc_pair_omegas(m.ptr, _p(cov6), len(cov6), _p(rel64), _p(corr), _p(om))
    return om


def pair_loglik_frozen(m: Map, mean3, rel64, corr, omega9) -> float:
    mean3 = _c(mean3, np.float32).reshape(-1, 3)
    rel64 = _c(np.asarray(rel64).reshape(12), np.float64)
    corr = _c(corr, np.int32)
    omega9 = _c(omega9, np.float64)
    return float(lib().orc_pair_loglik_frozen(m.ptr, _p(mean3), len(mean3), _p(rel64),
                                              _p(corr), _p(omega9)))


def gn_step(H, b, damping_rel=1e-6, step_clamp=1.0):
    H = _c(np.asarray(H).reshape(36), np.float64)
    b = _c(b, np.float64)
    psi = np.zeros(6, np.float64)
    cl = C.c_int32()
    rc = lib().orc_gn_step(_p(H), _p(b), damping_rel, step_clamp, _p(psi), C.byref(cl))
    return psi, bool(rc), bool(cl.value)


def propagation_ratio(D, t_o: int, D_now: float):
    D = _c(D, np.float64)
    r = np.zeros(len(D), np.float64)
    rc = lib().orc_propagation_ratio(_p(D), len(D), int(t_o), float(D_now), _p(r))
    return None if rc else r[: len(D) - t_o]


# ---------------------------------------------------------------- filter steps
def weights(L, l=None):
    L = _c(L, np.float64).copy()
    N = len(L)
    e = np.zeros(N, np.float64)
    w = np.zeros(N, np.float64)
    m = C.c_double()
    S = C.c_double()
    lib().orc_weights(N, _p(L), _p(None if l is None else _c(l, np.float64)), _p(e), _p(w),
                      C.byref(m), C.byref(S))
    return L, e, w, m.value, S.value


def dead(l, w, rel_floor=LN_1E16, post_floor=1e-8):
    l = _c(l, np.float64)
    w = _c(w, np.float64)
    d = np.zeros(len(l), np.uint8)
    nd = lib().orc_dead(len(l), _p(l), _p(w), rel_floor, post_floor, _p(d))
    return d, int(nd)


def resample(e, dead_mask, U: int):
    e = _c(e, np.float64)
    dm = _c(dead_mask, np.uint8)
    donor = np.zeros(len(e), np.int32)
    rc = lib().orc_resample(len(e), _p(e), _p(dm), int(U) & 0xFFFFFFFF, _p(donor))
    if rc:
        raise RuntimeError("degenerate: every particle dead")
    return donor


def diversity(t, h: float):
    """R35: d_i = (2 / (h N)) sum_j (t_i - t_j) exp(-|t_i - t_j|^2 / h) for translations t (N, 3)."""
    t = _c(np.asarray(t, np.float64).reshape(-1, 3), np.float64)
    d = np.zeros_like(t)
    lib().orc_diversity(len(t), _p(t), float(h), _p(d))
    return d


def representative(w) -> int:
    w = _c(w, np.float64)
    return int(lib().orc_representative(len(w), _p(w)))


def philox4x32_10(ctr, key):
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def normals8(seed: int, frame: int, gi: int):
    z = np.zeros(8)
    lib().orc_normals8(int(seed), int(frame), int(gi), _p(z))
    return z


def predict(pose12, dT12, cov36, seed: int, frame: int, gbase: int = 0, vertical_sigma=0.0):
    """Eq.1 prediction, in place on pose12 (N, 12) fp32."""
    assert pose12.dtype == np.float32 and pose12.flags.c_contiguous
    dT = _c(np.asarray(dT12).reshape(12), np.float32)
    cv = _c(np.asarray(cov36).reshape(36), np.float64)
    rc = lib().orc_predict(len(pose12), _p(pose12), _p(dT), _p(cv), int(seed), int(frame),
                           int(gbase), float(vertical_sigma))
    if rc:
        raise ValueError("covariance neither SPD nor zero")


def overlap(m: "Map", mean3, rel32) -> float:
    mean3 = _c(mean3, np.float32).reshape(-1, 3)
    r = _c(np.asarray(rel32).reshape(12), np.float32)
    return float(lib().orc_overlap(m.ptr, _p(mean3), len(mean3), _p(r)))


class Keyframes:
    """Oracle-side keyframe store: maps + shared path lengths D_k (R14)."""

    def __init__(self, clouds, D, r: float):
        self.maps = [Map(m3, c6, r) for (m3, c6) in clouds]
        self.D = _c(D, np.float64)
        self._ptrs = (C.c_void_p * len(self.maps))(*[m.ptr for m in self.maps])

    @property
    def K(self):
        return len(self.maps)

    def append(self, mean3, cov6, D_k: float, r: float):
        """Register one more keyframe."""
        self.maps.append(Map(mean3, cov6, r))
        self.D = np.append(self.D, float(D_k))
        self._ptrs = (C.c_void_p * len(self.maps))(*[m.ptr for m in self.maps])


def particles(cfg: Config, kfs: Keyframes, D_now, pose12, kf_pose12, scan_mean3, scan_cov6,
              idx=None, apply_update=True, slots=False):
    """Steps 2-7 on the particles idx (None = all); poses updated in place when apply_update."""
    pose12 = np.asarray(pose12)
    kf_pose12 = np.asarray(kf_pose12)
    assert pose12.dtype == np.float32 and pose12.flags.c_contiguous
    assert kf_pose12.dtype == np.float32 and kf_pose12.flags.c_contiguous
    N = pose12.reshape(-1, 12).shape[0]
    kf_stride = kf_pose12.reshape(N, -1, 12).shape[1]
    scan_mean3 = _c(scan_mean3, np.float32)
    scan_cov6 = _c(scan_cov6, np.float32)
    S = scan_mean3.reshape(-1, 3).shape[0]
    if idx is not None:
        idx = _c(idx, np.int32)
    n = N if idx is None else len(idx)
    nb = cfg.neighbor_count
    out = {"loglik": np.zeros(n), "grad6": np.zeros((n, 6)), "hess36": np.zeros((n, 6, 6)),
           "psi6": np.zeros((n, 6)), "flags": np.zeros(n, np.uint8)}
    if slots:
        out.update(slot_l=np.zeros((n, nb)), slot_H36=np.zeros((n, nb, 6, 6)),
                   slot_b6=np.zeros((n, nb, 6)), slot_n=np.zeros((n, nb), np.int32),
                   slot_kf=np.full((n, nb), -1, np.int32))
    po = ParticleOut(*[out[k].ctypes.data if k in out else None for k, _ in ParticleOut._fields_])
    rc = lib().orc_particles(C.byref(cfg), kfs.K, kfs._ptrs, _p(kfs.D), float(D_now), N,
                             _p(pose12), _p(kf_pose12), kf_stride, _p(scan_mean3),
                             _p(scan_cov6), S, _p(idx), n, int(bool(apply_update)), C.byref(po))
    if rc:
        raise RuntimeError(f"orc_particles rc={rc}")
    return out


def update(cfg: Config, kfs: Keyframes, D_now, pose12, kf_pose12, L, scan_mean3, scan_cov6, U):
    """The whole update (steps 2-11); pose12 / kf_pose12 / L updated in place."""
    pose12 = np.asarray(pose12)
    kf_pose12 = np.asarray(kf_pose12)
    assert pose12.dtype == np.float32 and kf_pose12.dtype == np.float32
    assert L.dtype == np.float64 and L.flags.c_contiguous
    N = pose12.reshape(-1, 12).shape[0]
    kf_stride = kf_pose12.reshape(N, -1, 12).shape[1]
    scan_mean3 = _c(scan_mean3, np.float32)
    scan_cov6 = _c(scan_cov6, np.float32)
    S = scan_mean3.reshape(-1, 3).shape[0]
    out = {"loglik": np.zeros(N), "grad6": np.zeros((N, 6)), "hess36": np.zeros((N, 6, 6)),
           "psi6": np.zeros((N, 6)), "weight": np.zeros(N), "donor": np.zeros(N, np.int32),
           "flags": np.zeros(N, np.uint8), "representative": np.zeros(1, np.int32),
           "n_dead": np.zeros(1, np.int64)}
    uo = UpdateOut(*[out[k].ctypes.data for k, _ in UpdateOut._fields_])
    rc = lib().orc_update(C.byref(cfg), kfs.K, kfs._ptrs, _p(kfs.D), float(D_now), N,
                          _p(pose12), _p(kf_pose12), kf_stride, _p(L), _p(scan_mean3),
                          _p(scan_cov6), S, int(U) & 0xFFFFFFFF, C.byref(uo))
    out["status"] = rc
    out["representative"] = int(out["representative"][0])
    out["n_dead"] = int(out["n_dead"][0])
    return out
