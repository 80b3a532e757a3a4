"""Shared comparison helpers for the GPU parity tests (CUDA product vs FP64 oracle)."""
from __future__ import annotations

import numpy as np

from paper_2404_03202_b200 import native

IMAGE_ATOL = 1e-4          # north_star: rendered images within 1e-4 absolute
GRAD_RTOL = 1e-3           # north_star: gradients within 1e-3 relative
GRAD_FLOOR = 1e-4          # abs floor, as a fraction of the group's max |grad| (norm-relative)


def gpu_tile_lists(frame: native.Frame):
    tx, ty, ranges, ids = frame.tiles()
    return [ids[r[0]:r[1]].astype(np.int64) for r in ranges]


def oracle_tile_lists(of):
    return [np.asarray(l, dtype=np.int64) for l in of.tile_gaussian_lists()]


def compare_tiles(frame, of):
    """Returns (n_tiles_mismatched, first_mismatch_tile)."""
    g = gpu_tile_lists(frame)
    o = oracle_tile_lists(of)
    assert len(g) == len(o), (len(g), len(o))
    bad = [t for t in range(len(g)) if not np.array_equal(g[t], o[t])]
    return len(bad), (bad[0] if bad else None)


def compare_projections(frame, of, n):
    pr = frame.projections()
    vis_o = np.zeros(n, dtype=bool)
    vis_o[of.gaussian_id] = True
    assert np.array_equal(pr["visible"], vis_o), "visible sets differ"
    gid = of.gaussian_id
    rel = lambda a, b: np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) if a.size else 0.0
    out = dict(
        p_abs=float(np.max(np.abs(pr["p"][gid] - of.p))) if gid.size else 0.0,
        conic_rel=rel(pr["conic"][gid], of.conic),
        opacity_rel=rel(pr["opacity"][gid], of.alpha),
        color_abs=float(np.max(np.abs(pr["color"][gid] - of.color))) if gid.size else 0.0,
    )
    # tile rect from the oracle's projection (rasterizer.cpp:67-78)
    ty_n, tx_n = of.tiles_y, of.tiles_x
    y0 = np.floor((of.p[:, 1] - of.radius) / 16).astype(np.int64)
    y1 = np.floor((of.p[:, 1] + of.radius) / 16).astype(np.int64)
    x0 = np.floor((of.p[:, 0] - of.radius) / 16).astype(np.int64)
    x1 = np.floor((of.p[:, 0] + of.radius) / 16).astype(np.int64)
    ty0, ty1 = np.maximum(y0, 0), np.minimum(y1, ty_n - 1)
    whole = (x1 - x0 + 1) >= tx_n
    x0 = np.where(whole, 0, x0)
    x1 = np.where(whole, tx_n - 1, x1)
    touched = np.where(ty0 > ty1, 0, (ty1 - ty0 + 1) * (x1 - x0 + 1))
    out["touched_mismatch"] = int(np.sum(pr["touched"][gid].astype(np.int64) != touched))
    return out


def grads_close(g_gpu: dict, g_or, groups=("d_position", "d_sh", "d_rotation", "d_log_scale", "d_opacity_logit")):
    """Per group: (entries outside the bar, total, max error / group scale, worst entry).

    The bar (north_star "gradients within 1e-3 relative"): |gpu - ref| <= 1e-3 max(|gpu|, |ref|),
    with an absolute floor of 1e-4 x the group's largest |ref| for entries that are themselves
    ~zero (a relative bar is undefined there). Tests require 0 entries outside the bar."""
    report = {}
    for k in groups:
        a = np.asarray(g_gpu[k], dtype=np.float64).ravel()
        b = np.asarray(getattr(g_or, k), dtype=np.float64).ravel()
        scale = max(np.max(np.abs(b)), 1e-30) if b.size else 1.0
        tol = np.maximum(GRAD_RTOL * np.maximum(np.abs(a), np.abs(b)), GRAD_FLOOR * scale)
        err = np.abs(a - b)
        bad = err > tol
        worst = int(np.argmax(err / tol)) if a.size else 0
        report[k] = (int(bad.sum()), a.size, float(np.max(err) / scale) if a.size else 0.0,
                     (worst, float(a[worst]), float(b[worst])) if a.size else None)
    return report


def assert_grads_close(g_gpu: dict, g_or, **kw):
    for k, (nbad, total, max_over_scale, worst) in grads_close(g_gpu, g_or, **kw).items():
        assert nbad == 0, f"{k}: {nbad}/{total} entries outside 1e-3 rel (max err/scale {max_over_scale:.2e}, " \
                          f"worst (index, gpu, ref) {worst})"
