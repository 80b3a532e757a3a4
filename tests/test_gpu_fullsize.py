"""GPU: element-wise parity at the BASELINE.json sizes against the reference's own code
(oracle/_ref, the reference sources compiled by oracle/Makefile, all host threads).

Every case compares, on identical FP32-representable inputs:
* tile lists (sorted keys / per-tile ranges) — bit-exact, every tile (rasterizer.cpp:57-98);
* contributors and last_contrib — exactly equal; image within 1e-4 absolute; T (rasterizer.cpp:100-157);
* the backward for the reference loss gradient (L1 + SSIM, lambda 0.2, of the oracle's own render
  against a seed-2 target) — every gradient entry within 1e-3 relative (tests/parity.py; no
  outlier allowance), screen_hits exactly, d_screen (gradients.cpp:72-296).

Cases (BASELINE configs[2] / [3] and the north_star's pole/seam views):
1M / 2048x1024 uniform (ring pose), pole-heavy (|lat| > 70 deg), seam-heavy (|lon| > 160 deg);
a near-opaque 1M scene (opacity U[0.95, 0.999]) that exercises the T < 1e-4 stop and the 0.99 clamp
gate; oversized near-opaque pole splats; 3M / 4096x2048. Measured errors of these cases:
profiles/parity_fullsize_r02.json.
"""
import os

import numpy as np
import pytest

from paper_2404_03202_b200 import native, scenes

from parity import IMAGE_ATOL, assert_grads_close, compare_tiles

pytestmark = pytest.mark.gpu

RING3 = scenes.ring_poses(16, seed=2)[3]
CASES = [
    # (id, cloud factory, pose, W, H)
    ("1m_uniform", lambda: scenes.synthetic_cloud(1_000_000, seed=1), RING3, 2048, 1024),
    ("1m_pole", lambda: scenes.synthetic_cloud(1_000_000, seed=1, variant="pole"), scenes.identity_pose(), 2048, 1024),
    ("1m_seam", lambda: scenes.synthetic_cloud(1_000_000, seed=1, variant="seam"), scenes.identity_pose(), 2048, 1024),
    ("1m_opaque", lambda: scenes.synthetic_cloud(1_000_000, seed=4, opacity_range=(0.95, 0.999)), RING3, 2048, 1024),
    ("opaque_pole_x1.5", lambda: scenes.synthetic_cloud(200_000, seed=3, variant="pole", opacity_range=(0.95, 0.999),
                                                        scale_mult=1.5), scenes.identity_pose(), 2048, 1024),
    ("3m_4096", lambda: scenes.synthetic_cloud(3_000_000, seed=1), RING3, 4096, 2048),
]


@pytest.fixture(scope="module")
def ref(oracle_ref):
    oracle_ref.set_threads(os.cpu_count() or 1)
    return oracle_ref


@pytest.mark.parametrize("name,make,pose,W,H", CASES, ids=[c[0] for c in CASES])
def test_full_size_matches_reference(name, make, pose, W, H, ref):
    cloud = make()
    ctx = native.Context(cloud)
    fr = ctx.render(pose, W, H)
    of = ref.render(cloud, pose, W, H, keep_handle=True)
    try:
        nbad, first = compare_tiles(fr, of)
        assert nbad == 0, f"{nbad} tile lists differ (first {first})"
        rgb, T, con, last = fr.pixels()
        assert np.array_equal(last, of.last_contrib), int(np.sum(last != of.last_contrib))
        assert np.array_equal(con, of.contributors), int(np.sum(con != of.contributors))
        err = float(np.max(np.abs(fr.image() - of.rgb)))
        assert err <= IMAGE_ATOL, err
        assert float(np.max(np.abs(T - of.T))) < 1e-5
        # the reference loss gradient of its own render against a different scene's render
        tctx = native.Context(scenes.synthetic_cloud(cloud.n, seed=cloud.n % 7 + 2))
        tf = tctx.render(pose, W, H)
        target = tf.image()
        tf.free()
        tctx.free()
        _, d_image = ref.loss(of.rgb, target, 0.2, 0.0)
        go = ref.backward(of, d_image, cloud, pose)
    finally:
        ref.free(of)
    ctx.backward(fr, d_image)
    g = ctx.gradients()
    fr.free()
    ctx.free()
    assert_grads_close(g, go)
    assert np.array_equal(g["screen_hits"], go.screen_hits)
    ds = np.max(np.abs(go.d_screen))
    assert np.max(np.abs(g["d_screen"] - go.d_screen)) <= 1e-3 * ds


def test_full_size_render_is_deterministic():
    """Bit-identical frames for the same inputs (test_rasterizer.cpp:151-169 through the GPU)."""
    cloud = scenes.synthetic_cloud(1_000_000, seed=1, variant="pole")
    ctx = native.Context(cloud)
    a = ctx.render(RING3, 2048, 1024)
    img = a.image()
    pix = a.pixels()
    a.free()
    b = ctx.render(RING3, 2048, 1024)
    assert np.array_equal(img, b.image())
    for x, y in zip(pix, b.pixels()):
        assert np.array_equal(x, y)


def test_full_size_backward_is_linear():
    """grad(a d1 + b d2) = a grad(d1) + b grad(d2) at 1M / 2048x1024 within FP32 noise."""
    W, H = 2048, 1024
    ctx = native.Context(scenes.synthetic_cloud(1_000_000, seed=1))
    pose = scenes.identity_pose()
    rng = np.random.default_rng(1)
    d1 = rng.uniform(-1, 1, size=(H, W, 3)) / (W * H)
    d2 = rng.uniform(-1, 1, size=(H, W, 3)) / (W * H)
    out = []
    fr = ctx.render(pose, W, H)
    for d in (d1, d2, 0.5 * d1 - 2.0 * d2):
        ctx.backward(fr, d)
        out.append(ctx.gradients())
    fr.free()
    g1, g2, g3 = out
    for k in ("d_position", "d_sh", "d_rotation", "d_log_scale", "d_opacity_logit"):
        lin = 0.5 * g1[k] - 2.0 * g2[k]
        scale = np.max(np.abs(lin))
        assert np.max(np.abs(g3[k] - lin)) <= 1e-3 * scale, k


def test_config2_scale_matches_reference(ref):
    """configs[1] scale (100k Gaussians, 1024x512, ring pose) with a random d_image."""
    cloud = scenes.synthetic_cloud(100_000, seed=2)
    pose = scenes.ring_poses(16, seed=2)[5]
    Wc, Hc = 1024, 512
    ctx = native.Context(cloud)
    fr = ctx.render(pose, Wc, Hc)
    of = ref.render(cloud, pose, Wc, Hc, keep_handle=True)
    nbad, first = compare_tiles(fr, of)
    assert nbad == 0, (nbad, first)
    rgb, T, con, last = fr.pixels()
    assert np.array_equal(last, of.last_contrib) and np.array_equal(con, of.contributors)
    assert np.max(np.abs(fr.image() - of.rgb)) <= IMAGE_ATOL
    d = np.random.default_rng(7).uniform(-1, 1, size=(Hc, Wc, 3)) / (Wc * Hc)
    ctx.backward(fr, d)
    g = ctx.gradients()
    go = ref.backward(of, d, cloud, pose)
    ref.free(of)
    assert_grads_close(g, go)


@pytest.mark.parametrize("name,make,pose,W,H", CASES[:5], ids=[c[0] for c in CASES[:5]])
def test_default_guard_band_equals_strict_bound(name, make, pose, W, H):
    """K3's default T-stop guard (a fixed relative 2^-10 band) against the strict mode, whose band
    is a rigorous bound on the FP32 transmittance error: identical stop decisions
    — contributors and last_contrib equal for every pixel — so on these scenes the default made every
    stop decision the FP64 reference makes (colours / T differ only where strict mode continued a
    pixel in FP64)."""
    cloud = make()
    out = []
    for strict in (False, True):
        ctx = native.Context(cloud)
        ctx.set_strict_guard(strict)
        fr = ctx.render(pose, W, H)
        out.append(fr.pixels())
        fr.free()
        ctx.free()
    (rgb_a, T_a, con_a, last_a), (rgb_b, T_b, con_b, last_b) = out
    assert np.array_equal(con_a, con_b) and np.array_equal(last_a, last_b)
    assert np.max(np.abs(rgb_a - rgb_b)) < 1e-5 and np.max(np.abs(T_a - T_b)) < 1e-5
