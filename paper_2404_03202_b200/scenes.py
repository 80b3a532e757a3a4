"""Deterministic synthetic scenes and poses (host-side data generation, numpy only).

Two generators:

* :func:`synthetic_cloud` — the benchmark scene of SURVEY.md §8(d): Gaussians on a shell
  r in [1.5, 2.5) around the origin, sigma_N = sqrt(53 / N) m, opacity U[0.05, 0.95),
  SH degree 3 (DC U[-0.4, 0.4), rest U[-0.1, 0.1)); variants ``uniform``, ``pole``
  (|lat| > 70 deg) and ``seam`` (|lon| > 160 deg).
* :func:`random_cloud` — the reference's own test scene (proj/tests/test_utils.hpp:52-90,
  ``CloudSpec``/``random_cloud``), same parameter ranges, numpy RNG.

Every parameter is rounded to float32 before either side sees it, so the FP64 oracle and the
FP32-resident device copy start from identical values.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Cloud:
    """Host mirror of the reference ``GaussianCloud`` (proj/include/omnisplat/scene.hpp:31-55).

    Arrays are float64 holding float32-representable values:
    positions (n,3), sh (n, bc, 3), rotations (n,4) raw (w,x,y,z), log_scales (n,3),
    opacity_logits (n,).
    """

    positions: np.ndarray
    sh: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    opacity_logits: np.ndarray
    sh_degree: int = 3
    active_sh_degree: int = 3

    @property
    def n(self) -> int:
        return int(self.positions.shape[0])

    @property
    def basis_count(self) -> int:
        return (self.sh_degree + 1) ** 2

    def copy(self) -> "Cloud":
        return Cloud(self.positions.copy(), self.sh.copy(), self.rotations.copy(),
                     self.log_scales.copy(), self.opacity_logits.copy(), self.sh_degree,
                     self.active_sh_degree)

    def rounded(self) -> "Cloud":
        f = lambda a: np.ascontiguousarray(a, dtype=np.float32).astype(np.float64)
        return Cloud(f(self.positions), f(self.sh), f(self.rotations), f(self.log_scales),
                     f(self.opacity_logits), self.sh_degree, self.active_sh_degree)


def _logit(p):
    return np.log(p / (1.0 - p))


def _directions(rng: np.random.Generator, n: int, variant: str) -> np.ndarray:
    out = np.empty((0, 3))
    while out.shape[0] < n:
        d = rng.standard_normal((max(2 * (n - out.shape[0]), 1024), 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        if variant == "pole":
            lat = np.degrees(np.arcsin(np.clip(d[:, 1], -1, 1)))
            d = d[np.abs(lat) > 70.0]
        elif variant == "seam":
            lon = np.degrees(np.arctan2(d[:, 0], d[:, 2]))
            d = d[np.abs(lon) > 160.0]
        elif variant == "avoid_poles":
            d = d[np.sqrt(d[:, 0] ** 2 + d[:, 2] ** 2) >= 0.2]
        elif variant != "uniform":
            raise ValueError(f"unknown variant {variant!r}")
        out = np.concatenate([out, d])
    return out[:n]


def synthetic_cloud(n: int, seed: int = 1, variant: str = "uniform", sh_degree: int = 3,
                    opacity_range=(0.05, 0.95), scale_mult: float = 1.0) -> Cloud:
    """The §8(d) generator. `opacity_range` / `scale_mult` only reshape the same random draws
    (stress scenes: near-opaque splats for the T < 1e-4 stop, oversized pole splats)."""
    rng = np.random.default_rng(seed)
    bc = (sh_degree + 1) ** 2
    dirs = _directions(rng, n, variant)
    dist = rng.uniform(1.5, 2.5, size=(n, 1))
    positions = dirs * dist
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sigma = np.sqrt(53.0 / max(n, 1))
    base = np.log(scale_mult * sigma * rng.uniform(0.5, 1.5, size=(n, 1)))
    log_scales = base + 0.1 * rng.standard_normal((n, 3))
    opacity_logits = _logit(rng.uniform(opacity_range[0], opacity_range[1], size=n))
    sh = np.empty((n, bc, 3))
    sh[:, 0, :] = rng.uniform(-0.4, 0.4, size=(n, 3))
    if bc > 1:
        sh[:, 1:, :] = rng.uniform(-0.1, 0.1, size=(n, bc - 1, 3))
    return Cloud(positions, sh, q, log_scales, opacity_logits, sh_degree, sh_degree).rounded()


def random_cloud(rng: np.random.Generator, count: int = 10, sh_degree: int = 3, min_dist=1.5,
                 max_dist=2.5, min_scale=0.15, max_scale=0.5, min_opacity=0.3, max_opacity=0.85,
                 dc_range=0.4, rest_range=0.1, avoid_poles=True) -> Cloud:
    """``random_cloud`` of proj/tests/test_utils.hpp:64-90 (numpy RNG, float32-rounded)."""
    bc = (sh_degree + 1) ** 2
    dirs = _directions(rng, count, "avoid_poles" if avoid_poles else "uniform")
    positions = dirs * rng.uniform(min_dist, max_dist, size=(count, 1))
    q = rng.standard_normal((count, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ls = np.log(rng.uniform(min_scale, max_scale, size=(count, 1)))
    log_scales = ls + 0.1 * rng.standard_normal((count, 3))
    opacity_logits = _logit(rng.uniform(min_opacity, max_opacity, size=count))
    sh = np.empty((count, bc, 3))
    sh[:, 0, :] = rng.uniform(-dc_range, dc_range, size=(count, 3))
    if bc > 1:
        sh[:, 1:, :] = rng.uniform(-rest_range, rest_range, size=(count, bc - 1, 3))
    return Cloud(positions, sh, q, log_scales, opacity_logits, sh_degree, sh_degree).rounded()


# ---------------------------------------------------------------------------- poses

def rot_x(a: float) -> np.ndarray:
    c, s = np.cos(a), np.sin(a)
    return np.array([[1, 0, 0], [0, c, -s], [0, s, c]], dtype=np.float64)


def rot_y(a: float) -> np.ndarray:
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]], dtype=np.float64)


def rot_z(a: float) -> np.ndarray:
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]], dtype=np.float64)


def quat_to_rotation(q) -> np.ndarray:
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def pose12(rotation: np.ndarray, translation=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Pose as 12 doubles: row-major world->camera rotation then t_cw (camera.hpp:21-30)."""
    p = np.zeros(12)
    p[:9] = np.asarray(rotation, dtype=np.float64).reshape(9)
    p[9:] = translation
    return p


def identity_pose() -> np.ndarray:
    return pose12(np.eye(3))


def random_pose(rng: np.random.Generator, center_radius: float = 0.2) -> np.ndarray:
    """random_pose of proj/tests/test_utils.hpp:42-50."""
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    R = quat_to_rotation(q)
    c = rng.uniform(-center_radius, center_radius, size=3)
    return pose12(R, -(R @ c))


def ring_poses(count: int, seed: int = 2, radius: float = 0.2) -> list:
    """Poses on a horizontal ring: yaw U[0, 2pi), centre on a circle."""
    rng = np.random.default_rng(seed)
    out = []
    for k in range(count):
        yaw = rng.uniform(0.0, 2.0 * np.pi)
        ang = 2.0 * np.pi * k / max(count, 1)
        centre = np.array([radius * np.cos(ang), 0.0, radius * np.sin(ang)])
        R = rot_y(yaw)
        out.append(pose12(R, -(R @ centre)))
    return out


def pose_to_transform(p12: np.ndarray) -> np.ndarray:
    """Row-major 4x4 world->camera transform for the reference C ABI (capi.cpp:88-95)."""
    t = np.eye(4)
    t[:3, :3] = p12[:9].reshape(3, 3)
    t[:3, 3] = p12[9:]
    return t


# ---------------------------------------------------------------------------- roaming scene (C5)

def roaming_scene(n: int = 2_000_000, seed: int = 5, rooms: int = 3, sh_degree: int = 3) -> Cloud:
    """360Roam-style synthetic interior: `rooms` connected 6 x 3 x 6 m rooms
    in a row along +x (y up, floor at y = 0), Gaussians as flat discs on the walls / floor /
    ceiling with procedural colour patterns (no two walls alike), plus volumetric blobs
    (furniture) inside each room. Doorways (1.2 m wide, 2.2 m high) join neighbouring rooms."""
    rng = np.random.default_rng(seed)
    Lx, Ly, Lz = 6.0, 3.0, 6.0
    n_blob = n // 6
    n_surf = n - n_blob
    # surface area per room: floor + ceiling 2*36, walls 4*18 (shared walls once)
    pts, nrm = [], []
    per = n_surf // rooms
    for r in range(rooms):
        x0 = r * Lx
        u = rng.random((per, 2))
        face = rng.choice(6, size=per, p=np.array([36, 36, 18, 18, 18, 18]) / 144.0)
        p = np.zeros((per, 3))
        nv = np.zeros((per, 3))
        # 0 floor, 1 ceiling, 2 wall z=0, 3 wall z=Lz, 4 wall x=x0, 5 wall x=x0+Lx
        for f, (ax, val, nn) in enumerate([(1, 0.0, (0, 1, 0)), (1, Ly, (0, -1, 0)), (2, 0.0, (0, 0, 1)),
                                           (2, Lz, (0, 0, -1)), (0, x0, (1, 0, 0)), (0, x0 + Lx, (-1, 0, 0))]):
            m = face == f
            k = int(m.sum())
            if ax == 1:
                p[m] = np.stack([x0 + u[m, 0] * Lx, np.full(k, val), u[m, 1] * Lz], axis=1)
            elif ax == 2:
                p[m] = np.stack([x0 + u[m, 0] * Lx, u[m, 1] * Ly, np.full(k, val)], axis=1)
            else:
                p[m] = np.stack([np.full(k, val), u[m, 1] * Ly, u[m, 0] * Lz], axis=1)
            nv[m] = nn
        # doorways: drop wall points inside the openings between rooms
        door = (((face == 4) & (r > 0)) | ((face == 5) & (r < rooms - 1))) & (np.abs(p[:, 2] - Lz / 2) < 0.6) & \
               (p[:, 1] < 2.2)
        pts.append(p[~door])
        nrm.append(nv[~door])
    P = np.concatenate(pts)
    Nrm = np.concatenate(nrm)
    ns = P.shape[0]
    # blobs: clusters of small Gaussians (furniture / objects)
    centres = np.stack([rng.uniform(0.5, rooms * Lx - 0.5, 40), rng.uniform(0.2, 1.5, 40), rng.uniform(0.5, Lz - 0.5, 40)], 1)
    which = rng.integers(0, 40, n_blob)
    B = centres[which] + rng.standard_normal((n_blob, 3)) * rng.uniform(0.1, 0.4, (40, 1))[which]
    positions = np.concatenate([P, B])
    total = positions.shape[0]
    # surface discs: thin along the normal; rotation maps local z to the normal
    spacing = np.sqrt(rooms * 144.0 / max(ns, 1))
    ls = np.empty((total, 3))
    ls[:ns, :2] = np.log(spacing * rng.uniform(0.6, 1.2, (ns, 2)))
    ls[:ns, 2] = np.log(spacing * 0.1)
    ls[ns:] = np.log(rng.uniform(0.005, 0.02, (total - ns, 1))) + 0.1 * rng.standard_normal((total - ns, 3))
    q = np.zeros((total, 4))
    z = np.array([0.0, 0.0, 1.0])
    axis = np.cross(np.broadcast_to(z, Nrm.shape), Nrm)
    s = np.linalg.norm(axis, axis=1)
    c = Nrm @ z
    ang = np.arctan2(s, c)
    axis = np.where(s[:, None] > 1e-9, axis / np.maximum(s, 1e-12)[:, None], np.array([1.0, 0.0, 0.0]))
    q[:ns, 0] = np.cos(ang / 2)
    q[:ns, 1:] = axis * np.sin(ang / 2)[:, None]
    q[:ns] = q[:ns] * np.where(q[:ns, :1] < 0, -1, 1)
    qb = rng.standard_normal((total - ns, 4))
    q[ns:] = qb / np.linalg.norm(qb, axis=1, keepdims=True)
    # colour: per-face palettes modulated by stripes / checkers in world coordinates
    base = rng.uniform(0.15, 0.85, (64, 3))
    cell = (np.floor(positions[:, 0] / 0.75) + 7 * np.floor(positions[:, 1] / 0.5) + 13 * np.floor(positions[:, 2] / 0.75))
    col = base[cell.astype(np.int64) % 64]
    col = col * (0.8 + 0.2 * np.sin(positions[:, :1] * 9.0) * np.cos(positions[:, 2:] * 7.0))
    col[ns:] = base[(which * 7) % 64] * rng.uniform(0.7, 1.1, (total - ns, 1))
    bc = (sh_degree + 1) ** 2
    sh = np.zeros((total, bc, 3))
    sh[:, 0, :] = (np.clip(col, 0.02, 0.98) - 0.5) / 0.28209479177387814
    if bc > 1:
        sh[:, 1:4, :] = rng.uniform(-0.03, 0.03, (total, 3, 3))
    opacity = _logit(np.concatenate([rng.uniform(0.85, 0.99, ns), rng.uniform(0.4, 0.95, total - ns)]))
    return Cloud(positions, sh, q, ls, opacity, sh_degree, sh_degree).rounded()


def roaming_poses(count: int = 200, seed: int = 6, rooms: int = 3) -> list:
    """Panorama centres along a wandering path through the rooms at eye height (1.4-1.7 m), random
    yaw; world->camera poses (camera y up)."""
    rng = np.random.default_rng(seed)
    t = np.linspace(0.0, 1.0, count)
    x = 0.8 + t * (rooms * 6.0 - 1.6)
    z = 3.0 + 1.8 * np.sin(t * rooms * 2.0 * np.pi) + rng.uniform(-0.3, 0.3, count)
    y = rng.uniform(1.4, 1.7, count)
    out = []
    for k in range(count):
        R = rot_y(rng.uniform(0.0, 2.0 * np.pi))
        c = np.array([x[k], y[k], z[k]])
        out.append(pose12(R, -(R @ c)))
    return out


def init_from_points(points: np.ndarray, rgb: np.ndarray, sh_degree: int = 3) -> Cloud:
    """init_from_points (proj/src/scene.cpp:181-213): isotropic scale sqrt(mean of the 3 nearest
    squared distances), identity rotation, opacity 0.1, DC colour from the point colour."""
    from scipy.spatial import cKDTree

    n = points.shape[0]
    d, _ = cKDTree(points).query(points, k=4)
    mean_sq = np.mean(d[:, 1:] ** 2, axis=1) if n > 1 else np.zeros(n)
    ls = np.log(np.sqrt(np.maximum(mean_sq, 1e-7)))
    bc = (sh_degree + 1) ** 2
    sh = np.zeros((n, bc, 3))
    sh[:, 0, :] = (rgb - 0.5) / 0.28209479177387814
    q = np.zeros((n, 4))
    q[:, 0] = 1.0
    return Cloud(points.copy(), sh, q, np.repeat(ls[:, None], 3, axis=1), np.full(n, _logit(0.1)), sh_degree,
                 0).rounded()
