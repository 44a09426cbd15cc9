"""Thin ctypes binding of libmcs (include/mcs.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/``; this module never
computes anything itself and has no CPU fallback: if ``libmcs.so`` is missing or no
CUDA device is present, the calls fail loudly.

Arrays may be numpy arrays or torch tensors (CPU or CUDA); the synchronous calls
accept host or device memory (the library copies through unified addressing).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCS_LIB", os.path.join(_HERE, "libmcs.so"))
HEADER = os.path.join(os.path.dirname(_HERE), "include", "mcs.h")

ABI_VERSION = 1
MAX_NEIGHBORS = 4
STATUS = {0: "MCS_OK", 1: "MCS_E_INVALID_ARG", 2: "MCS_E_OUT_OF_MEMORY", 3: "MCS_E_CUDA",
          4: "MCS_E_NCCL", 5: "MCS_E_CAPACITY", 6: "MCS_E_STATE", 7: "MCS_E_DEGENERATE"}
FLAG_LOOP, FLAG_UPDATED, FLAG_SINGULAR, FLAG_DEAD, FLAG_CLAMPED = 1, 2, 4, 8, 16


class MCSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [
        ("abi_version", C.c_uint32),
        ("capacity_particles", C.c_int32),
        ("capacity_keyframes", C.c_int32),
        ("capacity_scan_points", C.c_int32),
        ("neighbor_count", C.c_int32),
        ("loop_recency_gap", C.c_int32),
        ("voxel_resolution", C.c_float),
        ("gn_slots", C.c_int32),
        ("damping_rel", C.c_double),
        ("step_clamp", C.c_double),
        ("unmatched_penalty", C.c_double),
        ("loglik_rel_floor", C.c_double),
        ("posterior_floor", C.c_double),
        ("device", C.c_int32),
        ("rank", C.c_int32),
        ("world_size", C.c_int32),
        ("nccl_unique_id", C.c_void_p),
        ("transport", C.c_void_p),
        ("gn_iterations", C.c_int32),
        ("weight_after_update", C.c_int32),
        ("corr_mode", C.c_int32),
        ("nn_radius", C.c_float),
        ("clone_split", C.c_int32),
        ("allocator", C.c_void_p),
        ("peer_migration", C.c_int32),
        ("point_splits", C.c_int32),
        ("graph_replay", C.c_int32),
        ("kf_table_mib", C.c_int32),
        ("diversity_weight", C.c_double),
        ("diversity_bandwidth", C.c_double),
    ]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class Allocator(C.Structure):
    """mcs_allocator (include/mcs.h): the device-memory hook."""
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", C.c_void_p)]


class TorchAllocator:
    """Routes every libmcs device buffer through PyTorch's caching allocator, on the stream the
    library passes (its context stream), so library and torch tensors share one memory pool."""

    def __init__(self, device=None):
        import torch
        self._torch = torch
        self.device = torch.cuda.current_device() if device is None else int(device)

        def _alloc(nbytes, stream, user):
            try:
                return torch.cuda.caching_allocator_alloc(int(nbytes), self.device,
                                                          int(stream or 0))
            except Exception:  # out of memory -> NULL -> MCS_E_OUT_OF_MEMORY
                return None

        def _free(ptr, stream, user):
            torch.cuda.caching_allocator_delete(int(ptr))

        self._fns = (ALLOC_FN(_alloc), FREE_FN(_free))
        self.struct = Allocator(self._fns[0], self._fns[1], None)

    @property
    def ptr(self):
        return C.cast(C.pointer(self.struct), C.c_void_p)


CORR_CELL, CORR_NN27 = 0, 1


class UpdateOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("loglik", "grad6", "hess21", "psi6", "weight", "donor",
                                          "flags", "representative", "n_dead")]


_lib = None


def load() -> C.CDLL:
    """Load libmcs.so (never builds implicitly on the product path; see build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2504_18056_b200.build` "
                          "(no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp, i32, u32, f64 = C.c_void_p, C.c_int32, C.c_uint32, C.c_double
    st = C.c_int
    sig = {
        "mcs_config_default": (None, [vp]),
        "mcs_create": (st, [vp, vp]),
        "mcs_destroy": (st, [vp]),
        "mcs_last_error": (C.c_char_p, [vp]),
        "mcs_set_stream": (st, [vp, vp]),
        "mcs_add_keyframe": (st, [vp, vp, vp, i32, f64, vp]),
        "mcs_set_particles": (st, [vp, i32, vp, vp, vp]),
        "mcs_get_particles": (st, [vp, vp, vp, vp, vp]),
        "mcs_get_sizes": (st, [vp, vp, vp]),
        "mcs_update": (st, [vp, vp, vp, i32, f64, u32, vp]),
        "mcs_update_async": (st, [vp, vp, vp, i32, f64, u32, vp, vp]),
        "mcs_eval": (st, [vp, vp, vp, i32, vp, vp, vp, vp, vp, vp]),
        "mcs_resample": (st, [vp, vp, vp, i32, u32, vp]),
        "mcs_snapshot": (st, [vp]),
        "mcs_restore": (st, [vp]),
        "mcs_state_bytes_per_particle": (C.c_size_t, [i32]),
        "mcs_set_profiling": (st, [vp, i32]),
        "mcs_get_phase_ms": (st, [vp, vp]),
        "mcs_plan_ladder": (st, [i32, vp, vp, u32, vp, vp, vp, vp, vp]),
        "mcs_nccl_unique_id": (st, [vp]),
        "mcs_predict": (st, [vp, vp, vp, C.c_uint64, C.c_uint64, f64]),
        "mcs_overlap": (st, [vp, vp, i32, vp, i32, vp]),
        "mcs_inproc_transport_create": (vp, [i32]),
        "mcs_inproc_transport_destroy": (None, [vp]),
        "mcs_plan_migration": (st, [i32, vp, vp, vp]),
        "mcs_peer_migration_state": (i32, [vp]),
        "mcs_graph_state": (i32, [vp]),
        "mcs_scan_nonplanar": (st, [vp, vp]),
        "mcs_get_global_pose": (i32, [vp, C.c_int64, vp]),
        "mcs_get_pose": (st, [vp, i32, vp]),
        "mcs_config_size": (C.c_size_t, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def header_symbols() -> list[str]:
    """Every entry point include/mcs.h declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"MCS_API\s+[\w\s\*]*?\b(mcs_\w+)\s*\(", txt)))


def default_config(**kw) -> Config:
    n = load().mcs_config_size()
    if C.sizeof(Config) != n:  # the ctypes mirror must match include/mcs.h exactly
        raise RuntimeError(f"mcs_config is {n} bytes in libmcs but {C.sizeof(Config)} in the "
                           "binding: rebuild libmcs or update mcs.Config")
    cfg = Config()
    load().mcs_config_default(C.byref(cfg))
    for k, v in kw.items():
        if not hasattr(cfg, k):
            raise TypeError(f"unknown config field {k}")
        setattr(cfg, k, v)
    return cfg


def state_bytes_per_particle(n_keyframes: int) -> int:
    return int(load().mcs_state_bytes_per_particle(int(n_keyframes)))


# ------------------------------------------------------------------ marshalling
def _ptr(a, dtype, shape_last=None):
    """(pointer, keepalive) of a contiguous numpy array / torch tensor of the given dtype."""
    if a is None:
        return None, None
    try:
        import torch
        if isinstance(a, torch.Tensor):
            tdt = {np.float32: torch.float32, np.float64: torch.float64, np.int32: torch.int32,
                   np.uint8: torch.uint8, np.int64: torch.int64}[dtype]
            if a.dtype != tdt or not a.is_contiguous():
                a = a.to(tdt).contiguous()
            return a.data_ptr(), a
    except ImportError:  # pragma: no cover
        pass
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data, arr


class Context:
    """One mcs_ctx: the device keyframe store + particle shard of one GPU."""

    def __init__(self, capacity_particles: int, capacity_keyframes: int,
                 capacity_scan_points: int, **cfg_kw):
        self._lib = load()
        self._keep = []
        tr = cfg_kw.pop("transport", None)
        nid = cfg_kw.pop("nccl_unique_id", None)
        al = cfg_kw.pop("allocator", None)
        if al is not None:
            self._keep.append(al)
            if isinstance(al, TorchAllocator):
                al = al.ptr
            elif isinstance(al, Allocator):
                al = C.cast(C.pointer(al), C.c_void_p)
            cfg_kw["allocator"] = al
        if tr is not None:
            cfg_kw["transport"] = tr.ptr if isinstance(tr, (InprocTransport,
                                                            TorchDistTransport)) else tr
            self._keep.append(tr)
        if nid is not None:
            idbuf = C.create_string_buffer(bytes(nid), 128)
            self._keep.append(idbuf)
            cfg_kw["nccl_unique_id"] = C.cast(idbuf, C.c_void_p)
        self.cfg = default_config(capacity_particles=capacity_particles,
                                  capacity_keyframes=capacity_keyframes,
                                  capacity_scan_points=capacity_scan_points, **cfg_kw)
        self._ctx = C.c_void_p()
        st = self._lib.mcs_create(C.byref(self.cfg), C.byref(self._ctx))
        if st:
            raise MCSError(st, self._lib.mcs_last_error(None).decode())

    # -------------------------------------------------------------- plumbing
    def _check(self, st):
        if st:
            raise MCSError(st, self._lib.mcs_last_error(self._ctx).decode())

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            self._lib.mcs_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def sizes(self):
        n, k = C.c_int32(), C.c_int32()
        self._check(self._lib.mcs_get_sizes(self._ctx, C.byref(n), C.byref(k)))
        return n.value, k.value

    def set_stream(self, stream):
        """stream: torch.cuda.Stream, raw cudaStream_t int, or None (library-owned)."""
        h = getattr(stream, "cuda_stream", stream)
        self._check(self._lib.mcs_set_stream(self._ctx, C.c_void_p(h) if h else None))

    # -------------------------------------------------------------- state
    def add_keyframe(self, mean3, cov6, path_length: float) -> int:
        pm, km = _ptr(mean3, np.float32)
        pc, kc = _ptr(cov6, np.float32)
        n = int(np.prod(km.shape)) // 3
        kid = C.c_int32()
        self._check(self._lib.mcs_add_keyframe(self._ctx, pm, pc, n, float(path_length),
                                               C.byref(kid)))
        return kid.value

    def set_particles(self, pose12, kf_pose12=None, cum_loglik=None):
        pp, kp = _ptr(pose12, np.float32)
        n = int(np.prod(kp.shape)) // 12
        pk, kk = _ptr(kf_pose12, np.float32)
        pl, kl = _ptr(cum_loglik, np.float64)
        self._check(self._lib.mcs_set_particles(self._ctx, n, pp, pk, pl))

    @property
    def peer_migration_state(self) -> int:
        """1 peer-direct migration, -1 packed exchange, 0 not decided yet."""
        return int(self._lib.mcs_peer_migration_state(self._ctx))

    def get_global_pose(self, global_index: int) -> np.ndarray:
        """Collective over ranks: the pose (12,) of the particle with this GLOBAL index, e.g.
        the update's representative, on every rank (mcs_get_global_pose)."""
        p = np.zeros(12, np.float32)
        self._check(self._lib.mcs_get_global_pose(self._ctx, int(global_index), p.ctypes.data))
        return p

    @property
    def graph_captured(self) -> bool:
        """True when the library replays a captured CUDA graph of the update body."""
        return bool(self._lib.mcs_graph_state(self._ctx))

    def scan_nonplanar(self) -> int:
        """Points of the last prepared scan whose covariance is not plane-form (0: the sweep's
        plane-form instantiation runs; R36, mcs_scan_nonplanar)."""
        n = C.c_int32(0)
        self._check(self._lib.mcs_scan_nonplanar(self._ctx, C.byref(n)))
        return int(n.value)

    def get_pose(self, index: int) -> np.ndarray:
        """One local particle's current pose (12,) fp32 [R|t] row-major (mcs_get_pose)."""
        p = np.zeros(12, np.float32)
        self._check(self._lib.mcs_get_pose(self._ctx, int(index), p.ctypes.data))
        return p

    def get_particles(self, kf: bool = True):
        """Current poses, cumulative log-likelihoods and weights (and, with kf, every keyframe
        pose of every particle: N x K x 48 bytes)."""
        n, K = self.sizes
        pose = np.zeros((n, 12), np.float32)
        kfp = np.zeros((n, K, 12), np.float32) if kf else None
        L = np.zeros(n, np.float64)
        w = np.zeros(n, np.float64)
        self._check(self._lib.mcs_get_particles(self._ctx, pose.ctypes.data,
                                                kfp.ctypes.data if kf else None,
                                                L.ctypes.data, w.ctypes.data))
        out = {"pose12": pose, "L": L, "weight": w}
        if kf:
            out["kf_pose12"] = kfp
        return out

    def snapshot(self):
        self._check(self._lib.mcs_snapshot(self._ctx))

    def restore(self):
        self._check(self._lib.mcs_restore(self._ctx))

    # -------------------------------------------------------------- hot path
    def update(self, scan_mean3, scan_cov6, D_now: float, U: int, outputs=None,
               raise_degenerate=True, out=None):
        """mcs_update; returns a dict of numpy outputs (host).  outputs: iterable of names
        among loglik, grad6, hess21, psi6, weight, donor, flags (default all).  out: optional
        dict name -> caller-owned host buffer (numpy array or CPU tensor, e.g. pinned, of the
        output's dtype and size) written in place instead of fresh arrays."""
        n, _ = self.sizes
        out = out or {}
        names = ("loglik", "grad6", "hess21", "psi6", "weight", "donor", "flags") \
            if outputs is None else tuple(outputs)
        names = tuple(dict.fromkeys(names + tuple(out)))
        shapes = {"loglik": ((n,), np.float64), "grad6": ((n, 6), np.float32),
                  "hess21": ((n, 21), np.float32), "psi6": ((n, 6), np.float32),
                  "weight": ((n,), np.float64), "donor": ((n,), np.int32),
                  "flags": ((n,), np.uint8)}
        res = {}
        for k in names:
            if k in out:
                a = out[k].numpy() if hasattr(out[k], "numpy") else out[k]
                if (a.dtype != shapes[k][1] or a.size != int(np.prod(shapes[k][0])) or
                        not a.flags.c_contiguous):
                    raise ValueError(f"out[{k!r}] must be a contiguous {shapes[k][1].__name__} "
                                     f"buffer of {int(np.prod(shapes[k][0]))} elements")
                res[k] = a.reshape(shapes[k][0])
            else:
                res[k] = np.zeros(*shapes[k])
        rep = np.zeros(1, np.int32)
        nd = np.zeros(1, np.int64)
        uo = UpdateOut(**{k: (res[k].ctypes.data if k in res else None)
                          for k in ("loglik", "grad6", "hess21", "psi6", "weight", "donor",
                                    "flags")},
                       representative=rep.ctypes.data, n_dead=nd.ctypes.data)
        pm, km = _ptr(scan_mean3, np.float32)
        pc, kc = _ptr(scan_cov6, np.float32)
        S = int(np.prod(km.shape)) // 3
        st = self._lib.mcs_update(self._ctx, pm, pc, S, float(D_now), int(U) & 0xFFFFFFFF,
                                  C.byref(uo))
        if st and (st != 7 or raise_degenerate):
            self._check(st)
        res["representative"] = int(rep[0])
        res["n_dead"] = int(nd[0])
        res["status"] = int(st)
        return res

    def update_async(self, d_scan_mean3, d_scan_cov6, D_now: float, U: int, out=None,
                     stream=None):
        """mcs_update_async with torch CUDA tensors; out: dict name -> CUDA tensor."""
        out = out or {}
        fields = {}
        for k in ("loglik", "grad6", "hess21", "psi6", "weight", "donor", "flags",
                  "representative", "n_dead"):
            fields[k] = out[k].data_ptr() if k in out else None
        uo = UpdateOut(**fields)
        S = d_scan_mean3.numel() // 3
        h = getattr(stream, "cuda_stream", stream)
        self._check(self._lib.mcs_update_async(self._ctx, d_scan_mean3.data_ptr(),
                                               d_scan_cov6.data_ptr(), S, float(D_now),
                                               int(U) & 0xFFFFFFFF, C.byref(uo),
                                               C.c_void_p(h) if h else None))

    def eval(self, scan_mean3, scan_cov6):
        """mcs_eval: per (particle, slot) l, H (body frame, upper 21), b, n, keyframe id."""
        n, _ = self.sizes
        nb = self.cfg.neighbor_count
        out = {"slot_loglik": np.zeros((n, nb)), "slot_H21": np.zeros((n, nb, 21), np.float32),
               "slot_b6": np.zeros((n, nb, 6), np.float32),
               "slot_n": np.zeros((n, nb), np.int32), "slot_kf": np.zeros((n, nb), np.int32),
               "loop": np.zeros(n, np.uint8)}
        pm, km = _ptr(scan_mean3, np.float32)
        pc, kc = _ptr(scan_cov6, np.float32)
        S = int(np.prod(km.shape)) // 3
        self._check(self._lib.mcs_eval(self._ctx, pm, pc, S, *[out[k].ctypes.data for k in (
            "slot_loglik", "slot_H21", "slot_b6", "slot_n", "slot_kf", "loop")]))
        return out

    def resample(self, e, dead, U: int):
        pe, ke = _ptr(e, np.float64)
        pd, kd = _ptr(dead, np.uint8)
        n = int(np.prod(ke.shape))
        donor = np.zeros(n, np.int32)
        self._check(self._lib.mcs_resample(self._ctx, pe, pd, n, int(U) & 0xFFFFFFFF,
                                           donor.ctypes.data))
        return donor

    def predict(self, dT12, cov36, seed: int, frame: int, vertical_sigma: float = 0.0):
        """Eq.1 prediction of every local particle (mcs_predict)."""
        pd, kd = _ptr(np.asarray(dT12, np.float32).reshape(12), np.float32)
        pc, kc = _ptr(np.asarray(cov36, np.float64).reshape(36), np.float64)
        self._check(self._lib.mcs_predict(self._ctx, pd, pc, int(seed), int(frame),
                                          float(vertical_sigma)))

    def overlap(self, scan_mean3, rel12, kf: int) -> float:
        """Keyframe-insertion overlap rate of a scan against keyframe kf (mcs_overlap)."""
        pm, km = _ptr(scan_mean3, np.float32)
        pr, kr = _ptr(np.asarray(rel12, np.float32).reshape(12), np.float32)
        out = C.c_double()
        self._check(self._lib.mcs_overlap(self._ctx, pm, int(np.prod(km.shape)) // 3, pr,
                                          int(kf), C.byref(out)))
        return out.value

    def set_profiling(self, on: bool = True):
        self._check(self._lib.mcs_set_profiling(self._ctx, int(on)))

    def phase_ms(self):
        ms = (C.c_float * 5)()
        self._check(self._lib.mcs_get_phase_ms(self._ctx, ms))
        return {"select": ms[0], "sweep": ms[1], "update": ms[2], "weights": ms[3],
                "total": ms[4]}


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0 creates it; broadcast it to the other ranks)."""
    buf = C.create_string_buffer(128)
    st = load().mcs_nccl_unique_id(buf)
    if st:
        raise MCSError(st, "libnccl.so.2 unavailable")
    return buf.raw


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                          C.c_int32)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.POINTER(C.c_void_p),
                           C.POINTER(C.c_size_t), C.POINTER(C.c_void_p), C.POINTER(C.c_size_t))


class Transport(C.Structure):
    """mcs_transport (include/mcs.h): host collectives for world_size > 1 without NCCL."""
    _fields_ = [("user", C.c_void_p), ("allreduce", ALLREDUCE_FN), ("allgather", ALLGATHER_FN),
                ("alltoallv", ALLTOALLV_FN)]


class TorchDistTransport:
    """mcs_transport over a torch.distributed process group with CPU tensors (e.g. gloo): one
    process per rank.  Reductions are allgathered and reduced in rank order, so results are
    bitwise independent of the backend's reduction tree."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self._dist, self._torch, self.group = dist, torch, group
        self.world = dist.get_world_size(group)

        def _gather(b: bytes):
            t = torch.frombuffer(bytearray(b), dtype=torch.uint8)
            out = [torch.empty_like(t) for _ in range(self.world)]
            dist.all_gather(out, t, group=group)
            return [o.numpy().tobytes() for o in out]

        def allreduce(user, rank, buf, n, dtype, op):
            try:
                nbytes = 8 * n
                parts = _gather(C.string_at(buf, nbytes))
                arrs = [np.frombuffer(p, np.float64 if dtype == 0 else np.int64) for p in parts]
                acc = arrs[0].copy()
                for a in arrs[1:]:
                    acc = np.maximum(acc, a) if op == 1 else acc + a
                C.memmove(buf, acc.ctypes.data, nbytes)
                return 0
            except Exception:  # surfaced as MCS_E_NCCL by the library
                return 1

        def allgather(user, rank, send, recv, nbytes):
            try:
                parts = _gather(C.string_at(send, nbytes))
                C.memmove(recv, b"".join(parts), nbytes * self.world)
                return 0
            except Exception:
                return 1

        def alltoallv(user, rank, send, send_bytes, recv, recv_bytes):
            try:
                reqs = []
                bufs = []
                for p in range(self.world):
                    if p == rank:
                        continue
                    if send_bytes[p]:
                        t = torch.frombuffer(bytearray(C.string_at(send[p], send_bytes[p])),
                                             dtype=torch.uint8)
                        reqs.append(dist.isend(t, p, group=group))
                    if recv_bytes[p]:
                        r = torch.empty(recv_bytes[p], dtype=torch.uint8)
                        bufs.append((p, r))
                        reqs.append(dist.irecv(r, p, group=group))
                for q in reqs:
                    q.wait()
                for p, r in bufs:
                    C.memmove(recv[p], r.numpy().ctypes.data, recv_bytes[p])
                if send_bytes[rank]:
                    C.memmove(recv[rank], send[rank], send_bytes[rank])
                return 0
            except Exception:
                return 1

        self._fns = (ALLREDUCE_FN(allreduce), ALLGATHER_FN(allgather), ALLTOALLV_FN(alltoallv))
        self.struct = Transport(None, *self._fns)

    @property
    def ptr(self):
        return C.cast(C.pointer(self.struct), C.c_void_p)


class InprocTransport:
    """In-process transport joining `world` contexts (one thread per rank) on one device."""

    def __init__(self, world: int):
        self.world = world
        self.ptr = load().mcs_inproc_transport_create(int(world))

    def close(self):
        if self.ptr:
            load().mcs_inproc_transport_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def plan_ladder(Q_per_rank, D_per_rank, u: int):
    """Host plan of the global respawn ladder (mcs_plan_ladder): per-rank offsets and clone counts."""
    Q = np.ascontiguousarray(Q_per_rank, np.uint64)
    D = np.ascontiguousarray(D_per_rank, np.int64)
    G = len(Q)
    qo = np.zeros(G, np.uint64)
    do = np.zeros(G, np.int64)
    cl = np.zeros(G, np.int64)
    qt = np.zeros(1, np.uint64)
    dt = np.zeros(1, np.int64)
    st = load().mcs_plan_ladder(G, Q.ctypes.data, D.ctypes.data, int(u) & 0xFFFFFFFF,
                                qo.ctypes.data, do.ctypes.data, cl.ctypes.data, qt.ctypes.data,
                                dt.ctypes.data)
    return {"status": int(st), "q_offset": qo, "d_offset": do, "clones": cl,
            "Q": int(qt[0]), "D": int(dt[0])}


def plan_migration(clones_per_rank, dead_per_rank):
    """send[src, dst] = clones made on rank src that fill dead slots on rank dst."""
    c = np.ascontiguousarray(clones_per_rank, np.int64)
    d = np.ascontiguousarray(dead_per_rank, np.int64)
    G = len(c)
    out = np.zeros((G, G), np.int64)
    st = load().mcs_plan_migration(G, c.ctypes.data, d.ctypes.data, out.ctypes.data)
    if st:
        raise MCSError(st, "invalid migration plan input")
    return out


def unpack_h21(h21):
    """(..., 21) upper-triangle rows -> (..., 6, 6) symmetric."""
    h21 = np.asarray(h21)
    out = np.zeros(h21.shape[:-1] + (6, 6), h21.dtype)
    k = 0
    for r in range(6):
        for c in range(r, 6):
            out[..., r, c] = h21[..., k]
            out[..., c, r] = h21[..., k]
            k += 1
    return out


LN_1E16 = math.log(1e-16)
