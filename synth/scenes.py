"""Seeded synthetic LiDAR-like scenes for the MCS hot path (test/bench input only).

This module is the ONE thing the oracle side and the CUDA side share: it makes
inputs and holds none of the method's arithmetic (no SE(3) exp/log, no
likelihood, no relative poses, no weights).  Poses are built from scipy
rotation vectors and plain 4x4 products; covariances follow the GICP
convention the paper cites as boundary inputs (R9).

Recipe:
  1. ray-cast analytic primitives (axis-aligned boxes, vertical cylinders, a
     ground plane) with a MID-360-like pattern: 360 deg x [-7, +52] deg,
     range 0.1-40 m, sigma_range = 0.01 m (sensor of P:202);
  2. voxel-downsample on the fp32 cell grid floor(p * (1/r)) — one point per cell;
  3. random-subsample to exactly the requested count;
  4. covariances from the k = 10 nearest neighbours, plane-regularised to
     eigenvalues (1, 1, 1e-3), i.e. Sigma = I - (1 - eps) n n^T.
Every random draw comes from a Philox stream keyed (seed, purpose).
"""
from __future__ import annotations

import functools
import zlib
from dataclasses import dataclass, field

import numpy as np
from scipy.spatial import cKDTree
from scipy.spatial.transform import Rotation

EPS_PLANE = 1e-3


def rng(seed: int, purpose: str) -> np.random.Generator:
    key = (int(seed) << 32) | zlib.crc32(purpose.encode())
    return np.random.Generator(np.random.Philox(key=key))


# ------------------------------------------------------------------ poses
def pose(rotvec=(0.0, 0.0, 0.0), t=(0.0, 0.0, 0.0)) -> np.ndarray:
    """4x4 fp64 pose from a rotation vector and a translation."""
    T = np.eye(4)
    T[:3, :3] = Rotation.from_rotvec(np.asarray(rotvec, np.float64)).as_matrix()
    T[:3, 3] = t
    return T


def perturb(T: np.ndarray, sig_t: float, sig_r: float, g: np.random.Generator, n: int):
    """n poses T @ [R(phi) | rho], rho ~ N(0, sig_t^2 I), phi ~ N(0, sig_r^2 I); (n, 4, 4)."""
    rho = g.normal(0.0, sig_t, (n, 3))
    phi = g.normal(0.0, sig_r, (n, 3))
    D = np.tile(np.eye(4), (n, 1, 1))
    D[:, :3, :3] = Rotation.from_rotvec(phi).as_matrix()
    D[:, :3, 3] = rho
    return T @ D if T.ndim == 3 else np.einsum("ij,njk->nik", T, D)


def to12(T: np.ndarray) -> np.ndarray:
    """(..., 4, 4) fp64 -> (..., 12) fp32 row-major [R|t]."""
    return np.ascontiguousarray(T[..., :3, :4].reshape(T.shape[:-2] + (12,)), dtype=np.float32)


# ------------------------------------------------------------------ primitives
@dataclass
class World:
    boxes: np.ndarray = field(default_factory=lambda: np.zeros((0, 2, 3)))   # (nb, lo/hi, xyz)
    cylinders: np.ndarray = field(default_factory=lambda: np.zeros((0, 5)))  # (x, y, radius, z0, z1)
    ground_z: float | None = None


def _ray_boxes(o, d, boxes, tbest, chunk=32768):
    """Slab test of every ray against every box (torch CPU, multi-threaded)."""
    if len(boxes) == 0:
        return tbest
    import torch
    lo = torch.from_numpy(np.ascontiguousarray(boxes[:, 0, :] - o, np.float32))[None]
    hi = torch.from_numpy(np.ascontiguousarray(boxes[:, 1, :] - o, np.float32))[None]
    out = torch.from_numpy(tbest)
    for s in range(0, len(d), chunk):
        dd = torch.from_numpy(np.ascontiguousarray(d[s:s + chunk], np.float32))
        dd = torch.where(dd.abs() < 1e-12, torch.full_like(dd, 1e-12), dd)
        inv = (1.0 / dd)[:, None, :]
        t1 = lo * inv
        t2 = hi * inv
        tmin = torch.minimum(t1, t2).amax(dim=2)
        tmax = torch.maximum(t1, t2).amin(dim=2)
        tmin = torch.where((tmax >= tmin) & (tmin > 1e-6), tmin, torch.full_like(tmin, np.inf))
        out[s:s + chunk] = torch.minimum(out[s:s + chunk], tmin.amin(dim=1).double())
    return out.numpy()


def _ray_cylinders(o, d, cyl, tbest, chunk=32768):
    """Vertical cylinders (x, y, radius, z0, z1): nearest entry of every ray (torch CPU)."""
    if len(cyl) == 0:
        return tbest
    import torch
    cx = torch.from_numpy(np.ascontiguousarray(cyl[:, 0] - o[0], np.float64))[None]
    cy = torch.from_numpy(np.ascontiguousarray(cyl[:, 1] - o[1], np.float64))[None]
    rad = torch.from_numpy(np.ascontiguousarray(cyl[:, 2], np.float64))[None]
    z0 = torch.from_numpy(np.ascontiguousarray(cyl[:, 3], np.float64))[None]
    z1 = torch.from_numpy(np.ascontiguousarray(cyl[:, 4], np.float64))[None]
    out = torch.from_numpy(tbest)
    for s in range(0, len(d), chunk):
        dd = torch.from_numpy(np.ascontiguousarray(d[s:s + chunk], np.float64))
        dx, dy, dz = dd[:, 0:1], dd[:, 1:2], dd[:, 2:3]
        a = dx * dx + dy * dy
        b = -2 * (cx * dx + cy * dy)            # origin at 0, cylinder centre at (cx, cy)
        c = cx * cx + cy * cy - rad * rad
        disc = b * b - 4 * a * c
        ok = (disc > 0) & (a > 1e-12)
        t = (-b - torch.sqrt(torch.clamp(disc, min=0))) / (2 * torch.clamp(a, min=1e-12))
        z = o[2] + t * dz
        hit = ok & (t > 1e-6) & (z >= z0) & (z <= z1)
        t = torch.where(hit, t, torch.full_like(t, np.inf))
        out[s:s + chunk] = torch.minimum(out[s:s + chunk], t.amin(dim=1))
    return out.numpy()


def raycast(world: World, T_sensor: np.ndarray, n_az: int, n_el: int, g: np.random.Generator,
            el_range=(-7.0, 52.0), rmin=0.1, rmax=40.0, sigma=0.01) -> np.ndarray:
    """World-frame hit points of a jittered MID-360-like ray pattern from T_sensor."""
    az = (np.arange(n_az) + g.random(n_az)) * (2 * np.pi / n_az)
    el = np.deg2rad(el_range[0] + (np.arange(n_el) + g.random(n_el)) *
                    ((el_range[1] - el_range[0]) / n_el))
    A, E = np.meshgrid(az, el, indexing="ij")
    ds = np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], -1).reshape(-1, 3)
    d = ds @ T_sensor[:3, :3].T
    o = T_sensor[:3, 3]
    t = np.full(len(d), np.inf)
    t = _ray_boxes(o, d, world.boxes, t)
    t = _ray_cylinders(o, d, world.cylinders, t)
    if world.ground_z is not None:
        tg = (world.ground_z - o[2]) / np.where(np.abs(d[:, 2]) < 1e-12, -1e-12, d[:, 2])
        t = np.where((tg > 1e-6) & (tg < t), tg, t)
    keep = (t >= rmin) & (t <= rmax)
    t = t[keep] + g.normal(0.0, sigma, keep.sum())
    return o + d[keep] * t[:, None]


# ------------------------------------------------------------------ cloud processing
def downsample(p32: np.ndarray, r: float, g: np.random.Generator) -> np.ndarray:
    """One point per fp32 cell floor(p * (1/r)) (same grid the map uses, R27)."""
    p32 = np.ascontiguousarray(p32, np.float32)
    perm = g.permutation(len(p32))
    p32 = p32[perm]
    cells = np.floor(p32 * np.float32(1.0 / r)).astype(np.int64)
    _, first = np.unique(cells, axis=0, return_index=True)
    return p32[np.sort(first)]


def covariances(p: np.ndarray, k: int = 10, eps: float = EPS_PLANE) -> np.ndarray:
    """Plane-regularised GICP covariances, (n, 6) fp32 (xx, xy, xz, yy, yz, zz)."""
    p = np.asarray(p, np.float64)
    tree = cKDTree(p)
    _, nn = tree.query(p, k=min(k, len(p)))
    Q = p[nn] - p[nn].mean(axis=1, keepdims=True)
    cov = np.einsum("nki,nkj->nij", Q, Q) / max(nn.shape[1] - 1, 1)
    _, vec = np.linalg.eigh(cov)
    n = vec[:, :, 0]  # smallest-eigenvalue direction = surface normal
    Sig = np.eye(3)[None] - (1.0 - eps) * np.einsum("ni,nj->nij", n, n)
    out = np.stack([Sig[:, 0, 0], Sig[:, 0, 1], Sig[:, 0, 2], Sig[:, 1, 1], Sig[:, 1, 2],
                    Sig[:, 2, 2]], -1)
    return np.ascontiguousarray(out, np.float32)


def sensor_cloud(world: World, T_sensor: np.ndarray, r: float, count: int | None,
                 g: np.random.Generator, n_az: int, n_el: int, crop_backward: bool = False):
    """Ray cast -> sensor frame -> (backward crop) -> downsample at r -> (subsample to
    count) -> covariances."""
    pw = raycast(world, T_sensor, n_az, n_el, g)
    Ti = np.linalg.inv(T_sensor)
    ps = (pw @ Ti[:3, :3].T + Ti[:3, 3]).astype(np.float32)
    if crop_backward:
        ps = ps[ps[:, 0] > 0]
    ds = downsample(ps, r, g)
    cov_all = covariances(ds)
    if count is not None:
        if len(ds) < count:
            raise ValueError(f"only {len(ds)} cells after downsampling, need {count}")
        sel = np.sort(g.choice(len(ds), count, replace=False))
        ds, cov_all = ds[sel], cov_all[sel]
    return np.ascontiguousarray(ds, np.float32), np.ascontiguousarray(cov_all, np.float32)


# ------------------------------------------------------------------ worlds
def _slab(lo, hi):
    return np.array([lo, hi], np.float64)


def box_room(seed: int) -> World:
    """20 x 10 x 3 m room (C1) with a few boxes inside to constrain every axis."""
    g = rng(seed, "box_room")
    w = 0.2
    boxes = [
        _slab([-w, -w, -w], [20 + w, 10 + w, 0]),       # floor
        _slab([-w, -w, 3], [20 + w, 10 + w, 3 + w]),    # ceiling
        _slab([-w, -w, 0], [0, 10 + w, 3]),             # walls
        _slab([20, -w, 0], [20 + w, 10 + w, 3]),
        _slab([-w, -w, 0], [20 + w, 0, 3]),
        _slab([-w, 10, 0], [20 + w, 10 + w, 3]),
    ]
    for _ in range(8):
        c = g.uniform([1, 1, 0], [19, 9, 0])
        s = g.uniform([0.4, 0.4, 0.5], [1.2, 1.2, 2.0])
        boxes.append(_slab([c[0], c[1], 0], [c[0] + s[0], c[1] + s[1], s[2]]))
    return World(boxes=np.array(boxes))


def loop_corridor(seed: int, outer=(60.0, 40.0), width=10.0, height=8.0, n_clutter=160) -> World:
    """Rectangular loop corridor, warehouse-sized: 60 x 40 m, 10 m wide, 8 m high,
    with wall-side clutter (shelves, crates) so every axis is constrained."""
    g = rng(seed, "loop_corridor")
    X, Y = outer
    w = 0.3
    boxes = [
        _slab([-w, -w, -w], [X + w, Y + w, 0]),
        _slab([-w, -w, height], [X + w, Y + w, height + w]),
        _slab([-w, -w, 0], [0, Y + w, height]),
        _slab([X, -w, 0], [X + w, Y + w, height]),
        _slab([-w, -w, 0], [X + w, 0, height]),
        _slab([-w, Y, 0], [X + w, Y + w, height]),
        _slab([width, width, 0], [X - width, Y - width, height]),  # inner block
    ]
    # clutter: boxes against the outer and inner walls, and a few pillars mid-corridor
    for _ in range(n_clutter):
        side = g.integers(0, 4)
        along = g.uniform(0.0, 1.0)
        s = g.uniform([0.3, 0.3, 0.4], [2.5, 2.0, 5.0])
        inner = g.random() < 0.5
        off = (width - s[1]) if inner else 0.0
        if side == 0:    # y = 0 side
            x, y = along * (X - s[0]), off
        elif side == 1:  # y = Y side
            x, y = along * (X - s[0]), Y - s[1] - off
        elif side == 2:  # x = 0 side
            x, y = off, along * (Y - s[0])
            s = s[[1, 0, 2]]
        else:            # x = X side
            x, y = X - s[1] - off, along * (Y - s[0])
            s = s[[1, 0, 2]]
        boxes.append(_slab([x, y, 0], [x + s[0], y + s[1], s[2]]))
    return World(boxes=np.array(boxes))


def loop_path(arc: float, outer=(60.0, 40.0), width=10.0, z=1.5) -> np.ndarray:
    """Pose on the corridor centre line at arc length `arc` (counter-clockwise), heading along it."""
    X, Y = outer
    h = width / 2
    L1, L2 = X - 2 * h, Y - 2 * h
    P = 2 * (L1 + L2)
    s = arc % P
    if s < L1:
        p, yaw = (h + s, h), 0.0
    elif s < L1 + L2:
        p, yaw = (X - h, h + s - L1), np.pi / 2
    elif s < 2 * L1 + L2:
        p, yaw = (X - h - (s - L1 - L2), Y - h), np.pi
    else:
        p, yaw = (h, Y - h - (s - 2 * L1 - L2)), 1.5 * np.pi
    return pose((0, 0, yaw), (p[0], p[1], z))


def loop_perimeter(outer=(60.0, 40.0), width=10.0) -> float:
    return 2 * ((outer[0] - width) + (outer[1] - width))


# ------------------------------------------------------------------ configs
@dataclass
class Scene:
    name: str
    r: float
    gap: int
    keyframes: list            # [(mean3 (n,3) f32, cov6 (n,6) f32)] in each keyframe's own frame
    D: np.ndarray              # (K,) f64 cumulative odometry path length at each keyframe
    D_now: float
    scan_mean3: np.ndarray     # (S, 3) f32, sensor frame
    scan_cov6: np.ndarray      # (S, 6) f32
    pose12: np.ndarray         # (N, 12) f32 current poses T_t^i
    kf_pose12: np.ndarray      # (N, K, 12) f32 per-particle keyframe poses T_k^i
    U: int                     # resampling uniform (uint32)
    T_gt: np.ndarray = None    # (4, 4) true scan pose
    kf_gt: np.ndarray = None   # (K, 4, 4) true keyframe poses

    @property
    def N(self):
        return self.pose12.shape[0]

    @property
    def K(self):
        return len(self.keyframes)

    @property
    def S(self):
        return self.scan_mean3.shape[0]


@functools.lru_cache(maxsize=8)
def c1(seed: int = 0, N: int = 1000, S: int = 512, n_kf_pts: int = 2048) -> Scene:
    """C1: box room (r = 0.25 m), 1 keyframe of 2,048 points, 512-point scan 0.3 m / 3 deg away, gap 0."""
    world = box_room(seed)
    r = 0.25
    T_kf = pose((0, 0, 0.3), (6.0, 4.5, 1.4))
    T_gt = T_kf @ pose(np.deg2rad([0.0, 0.0, 3.0]), (0.3, 0.0, 0.0))
    kf = sensor_cloud(world, T_kf, r, n_kf_pts, rng(seed, "c1/kf"), 720, 160)
    scan = sensor_cloud(world, T_gt, r, S, rng(seed, "c1/scan"), 720, 160)
    g = rng(seed, "c1/particles")
    Tt = perturb(T_gt, 0.1, 0.02, g, N)
    Tk = perturb(T_kf, 0.0, 0.0, g, N)[:, None]
    return Scene("C1", r, 0, [kf], np.array([0.0]), 0.3, scan[0], scan[1], to12(Tt), to12(Tk),
                 int(rng(seed, "c1/U").integers(0, 2**32)), T_gt, T_kf[None])


@functools.lru_cache(maxsize=4)
def c2(seed: int = 0, N: int = 100_000, S: int = 4096, K: int = 20, gap: int = 10,
       sig_t: float = 0.2, sig_r: float = 0.02, drift_t: float = 0.01, drift_r: float = 0.001,
       n_az: int = 900, n_el: int = 150) -> Scene:
    """C2: loop corridor, K keyframes around the loop, scan back near keyframe 1 after a lap.

    Every particle's neighbours {0, 1, 2} are old (<= latest - gap), so every particle
    takes the full loop path (a2-a4).  Keyframe clouds downsampled at r = 0.5 m; the
    scan at r/2 then subsampled to exactly S points.
    """
    world = loop_corridor(seed)
    r = 0.5
    P = loop_perimeter()
    D = np.arange(K) * (P / K)
    kf_gt = np.stack([loop_path(d) for d in D])
    kfs = [sensor_cloud(world, kf_gt[k], r, None, rng(seed, f"c2/kf{k}"), n_az, n_el)
           for k in range(K)]
    arc_now = P + D[1] + 0.4
    T_gt = loop_path(arc_now) @ pose((0.01, -0.01, 0.02), (0.0, 0.15, 0.0))
    scan = sensor_cloud(world, T_gt, r / 2, S, rng(seed, "c2/scan"), n_az, n_el)
    g = rng(seed, "c2/particles")
    Tt = perturb(T_gt, sig_t, sig_r, g, N)
    # per-particle keyframe poses: GT composed with a random-walk drift growing with k
    Tk = np.empty((N, K, 4, 4))
    drift = np.tile(np.eye(4), (N, 1, 1))
    for k in range(K):
        drift = perturb(drift, drift_t, drift_r, g, N) if k > 0 else drift
        Tk[:, k] = np.einsum("ij,njk->nik", kf_gt[k], drift)
    return Scene("C2", r, gap, kfs, D, float(P + D[1] + 0.4), scan[0], scan[1], to12(Tt),
                 to12(Tk), int(rng(seed, "c2/U").integers(0, 2**32)), T_gt, kf_gt)


def forest(seed: int, rows: int = 10, pitch: float = 5.0) -> World:
    """Forest-like grid: rows x rows trees at `pitch`, radius 0.3 +- 0.05 m, 8 m
    tall, on a ground plane — repeated geometry with one-pitch ambiguity."""
    g = rng(seed, "forest")
    xs = np.arange(rows) * pitch
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    n = rows * rows
    cyl = np.stack([X.ravel() + g.normal(0, 0.1, n), Y.ravel() + g.normal(0, 0.1, n),
                    0.3 + g.uniform(-0.05, 0.05, n), np.zeros(n), np.full(n, 8.0)], 1)
    return World(cylinders=cyl, ground_z=0.0)


def forest_path(arc: float, lo=2.5, hi=42.5, z=1.5) -> np.ndarray:
    """Counter-clockwise rectangular lap in the gaps between tree rows."""
    L = hi - lo
    s = arc % (4 * L)
    if s < L:
        p, yaw = (lo + s, lo), 0.0
    elif s < 2 * L:
        p, yaw = (hi, lo + s - L), np.pi / 2
    elif s < 3 * L:
        p, yaw = (hi - (s - 2 * L), hi), np.pi
    else:
        p, yaw = (lo, hi - (s - 3 * L)), 1.5 * np.pi
    return pose((0, 0, yaw), (p[0], p[1], z))


def _kf_poses_drift(kf_gt, N, g, drift_t, drift_r):
    """(N, K, 12) fp32: GT keyframe poses composed with a per-particle random-walk drift."""
    K = len(kf_gt)
    out = np.empty((N, K, 12), np.float32)
    drift = np.tile(np.eye(4), (N, 1, 1))
    for k in range(K):
        if k > 0:
            drift = perturb(drift, drift_t, drift_r, g, N)
        out[:, k] = to12(np.einsum("ij,njk->nik", kf_gt[k], drift))
    return out


@functools.lru_cache(maxsize=2)
def c3(seed: int = 0, N: int = 100_000, S: int = 4096, K: int = 200, gap: int = 10,
       modes=((0.0, 0.0), (5.0, 0.0), (-5.0, 0.0), (0.0, 5.0))) -> Scene:
    """C3: forest-like grid, r = 1 m, K keyframes from a prior lap (backward-cropped scans,
    P:168), the current scan back near the start; particles in lattice-shifted modes one tree
    pitch apart (the multimodal loop-closure ambiguity of P:168-170)."""
    world = forest(seed)
    r = 1.0
    L = 4 * 40.0
    D = np.arange(K) * (L / K)
    kf_gt = np.stack([forest_path(d) for d in D])
    kfs = [sensor_cloud(world, kf_gt[k], r, None, rng(seed, f"c3/kf{k}"), 512, 84,
                        crop_backward=True) for k in range(K)]
    T_gt = forest_path(L + D[2] + 0.3) @ pose((0.0, 0.0, 0.02), (0.0, 0.2, 0.0))
    scan = sensor_cloud(world, T_gt, r / 4, S, rng(seed, "c3/scan"), 1024, 168,
                        crop_backward=True)
    g = rng(seed, "c3/particles")
    per = -(-N // len(modes))
    Tt = np.concatenate([perturb(pose(t=(dx, dy, 0.0)) @ T_gt, 0.2, 0.02, g, per)
                         for dx, dy in modes])[:N]
    Tk = _kf_poses_drift(kf_gt, N, g, 0.005, 0.0005)
    return Scene("C3", r, gap, kfs, D, float(L + D[2] + 0.3), scan[0], scan[1], to12(Tt), Tk,
                 int(rng(seed, "c3/U").integers(0, 2**32)), T_gt, kf_gt)


def multi_floor(seed: int, floors: int = 2, height: float = 3.5) -> World:
    """Near-identical floors: one layout of walls and furniture repeated every
    `height` metres, plus one distinguishing box per floor."""
    base = loop_corridor(seed, outer=(30.0, 20.0), width=6.0, height=3.0, n_clutter=60)
    boxes = []
    for f in range(floors):
        off = np.array([0.0, 0.0, f * height])
        boxes.extend(list(base.boxes + off))
        c = rng(seed, f"floor{f}").uniform([2, 2, 0], [28, 4, 0]) + off
        boxes.append(np.array([c, c + [1.5, 1.5, 2.0]]))
    return World(boxes=np.array(boxes))


@functools.lru_cache(maxsize=2)
def c5(seed: int = 0, N: int = 100_000, S: int = 4096, K_floor: int = 20, gap: int = 10,
       height: float = 3.5) -> Scene:
    """C5: kidnapping across two floors.  Keyframes 0..K-1 from a lap of floor 1,
    K..2K-1 from the same lap on floor 2; the scan is on floor 2 after the elevator; particles
    spread vertically over both floors (the elevator's vertical random walk)."""
    world = multi_floor(seed, 2, height)
    r = 0.5
    P = 2 * ((30.0 - 6.0) + (20.0 - 6.0))
    path = lambda arc, f: loop_path(arc, outer=(30.0, 20.0), width=6.0, z=1.5 + f * height)
    D1 = np.arange(K_floor) * (P / K_floor)
    kf_gt = np.stack([path(d, 0) for d in D1] + [path(d, 1) for d in D1])
    D = np.concatenate([D1, P + 10.0 + D1])
    kfs = [sensor_cloud(world, kf_gt[k], r, None, rng(seed, f"c5/kf{k}"), 600, 100)
           for k in range(2 * K_floor)]
    T_gt = path(D1[1] + 0.3, 1)
    scan = sensor_cloud(world, T_gt, r / 2, S, rng(seed, "c5/scan"), 900, 150)
    g = rng(seed, "c5/particles")
    Tt = perturb(T_gt, 0.2, 0.02, g, N)
    Tt[:, 2, 3] += np.where(g.random(N) < 0.5, -height, 0.0) + g.normal(0, 0.3, N)
    Tk = _kf_poses_drift(kf_gt, N, g, 0.01, 0.001)
    D_now = float(2 * P + 20.0 + D1[1] + 0.3)
    return Scene("C5", r, gap, kfs, D, D_now, scan[0], scan[1], to12(Tt), Tk,
                 int(rng(seed, "c5/U").integers(0, 2**32)), T_gt, kf_gt)


@functools.lru_cache(maxsize=1)
def c4(seed: int = 0, N: int = 1_000_000, S: int = 8192, sig_t: float = 0.1, sig_r: float = 0.01,
       drift_t: float = 0.01, drift_r: float = 0.001) -> Scene:
    """C4: the C2 scene with an 8,192-point scan and 1M particles (sharded over 2/4/8 GPUs).
    A tighter spread (bench --config c4_survival) lets a share of the particles survive P:190's
    floors, so a6 clones (and, across GPUs, migrates) a realistic fraction."""
    base = c2(seed, N=1000)
    world = loop_corridor(seed)
    scan = sensor_cloud(world, base.T_gt, base.r / 2, S, rng(seed, "c4/scan"), 1200, 200)
    g = rng(seed, "c4/particles")
    Tt = perturb(base.T_gt, sig_t, sig_r, g, N)
    Tk = _kf_poses_drift(base.kf_gt, N, g, drift_t, drift_r)
    import dataclasses
    return dataclasses.replace(base, name="C4", scan_mean3=scan[0], scan_cov6=scan[1],
                               pose12=to12(Tt), kf_pose12=Tk,
                               U=int(rng(seed, "c4/U").integers(0, 2**32)))


def subset(scene: Scene, N: int) -> Scene:
    """The first N particles of a scene (same keyframes and scan)."""
    import dataclasses
    return dataclasses.replace(scene, pose12=np.ascontiguousarray(scene.pose12[:N]),
                               kf_pose12=np.ascontiguousarray(scene.kf_pose12[:N]))


# ------------------------------------------------------------------ trajectories (multi-frame)
@dataclass
class Trajectory:
    name: str
    r: float
    gap: int
    scans: list                # [(mean3 (S,3) f32, cov6 (S,6) f32)] in the sensor frame
    clouds: list               # [(mean3, cov6)] the whole frame downsampled at r (keyframe /
                               # overlap cloud)
    gt: np.ndarray             # (F, 4, 4) true sensor poses
    odom: np.ndarray           # (F, 4, 4) drifting odometry poses T^o_t
    odom_cov: np.ndarray       # (6, 6) covariance of one relative motion, twist order (rho, phi)
    D: np.ndarray              # (F,) cumulative odometry path length (R14)
    U: np.ndarray              # (F,) uint32 resampling uniforms

    @property
    def F(self):
        return len(self.scans)


def corridor_lap(seed: int = 0, n_frames: int = 90, step: float = 2.0, S: int = 1024,
                 r: float = 0.5, gap: int = 10, sig_t: float = 0.03, sig_r: float = 0.003,
                 n_az: int = 360, n_el: int = 64, arc0: float = 0.0) -> Trajectory:
    """A lap of the loop corridor (perimeter 160 m) and back past the start: GT poses every
    `step` metres, LiDAR-like scans at r/2 subsampled to S points, and an odometry whose every
    relative motion carries N(0, diag(sig_t^2 I, sig_r^2 I)) noise, so it drifts and the loop
    must be closed by the filter."""
    world = loop_corridor(seed)
    arcs = arc0 + step * np.arange(n_frames)
    gt = np.stack([loop_path(a) for a in arcs])
    g = rng(seed, "traj/odom")
    odom = np.empty_like(gt)
    odom[0] = gt[0]
    for k in range(1, n_frames):
        rel = np.linalg.inv(gt[k - 1]) @ gt[k]
        odom[k] = odom[k - 1] @ perturb(rel, sig_t, sig_r, g, 1)[0]
    scans, clouds = [], []
    for k in range(n_frames):
        g = rng(seed, f"traj/scan{k}")
        pw = raycast(world, gt[k], n_az, n_el, g)
        Ti = np.linalg.inv(gt[k])
        ps = (pw @ Ti[:3, :3].T + Ti[:3, 3]).astype(np.float32)
        full = downsample(ps, r, g)
        clouds.append((np.ascontiguousarray(full), covariances(full)))
        fine = downsample(ps, r / 2, g)
        sel = np.sort(g.choice(len(fine), S, replace=False))
        scans.append((np.ascontiguousarray(fine[sel]), covariances(fine)[sel]))
    D = np.concatenate([[0.0], np.cumsum(np.linalg.norm(np.diff(odom[:, :3, 3], axis=0),
                                                          axis=1))])
    cov = np.diag([sig_t ** 2] * 3 + [sig_r ** 2] * 3)
    U = rng(seed, "traj/U").integers(0, 2**32, n_frames).astype(np.uint32)
    return Trajectory("corridor_lap", r, gap, scans, clouds, gt, odom, cov, D, U)
