"""Synthetic host SplatProjection records (rasterizer.hpp:31-41) for the bin_to_tiles /
blend_forward-on-host-projections paths (osplat_gpu_render_projected, the compat shim)."""
import numpy as np


def random_splats(n: int, W: int, H: int, seed: int, ties: bool = True) -> dict:
    """n records over a W x H image: centres anywhere (seam and poles included), SPD covariances
    with conic = cov^-1 and radius = ceil(3 sqrt(lambda_max)) like project_gaussian, depths with
    deliberate ties (the (depth, gaussian_id) tie-break), shuffled gaussian ids, opacities up to
    1 (the 0.99 clamp)."""
    rng = np.random.default_rng(seed)
    p = np.stack([rng.uniform(-2.0, W + 2.0, n), rng.uniform(0.0, H, n)], axis=1)
    a = rng.uniform(0.5, 40.0, n)
    c = rng.uniform(0.5, 40.0, n)
    b = rng.uniform(-0.8, 0.8, n) * np.sqrt(a * c)
    cov = np.stack([a, b, c], axis=1)
    det = a * c - b * b
    conic = np.stack([c / det, -b / det, a / det], axis=1)
    mid = 0.5 * (a + c)
    dd = np.sqrt(np.maximum(0.25 * (a - c) ** 2 + b * b, 0.0))
    radius = np.ceil(3.0 * np.sqrt(mid + dd))
    depth = rng.uniform(1.0, 3.0, n)
    if ties and n >= 8:
        k = n // 4
        depth[rng.choice(n, k, replace=False)] = depth[rng.choice(n, k, replace=True)]
    return dict(gaussian_id=rng.permutation(n).astype(np.int32) * 3 + 1, p=p, cov=cov, conic=conic,
                radius=radius, depth=depth, color=rng.uniform(0.0, 1.0, (n, 3)),
                alpha_base=rng.uniform(0.02, 1.0, n))
