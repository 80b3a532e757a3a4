"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle on identical inputs.

Bars (BASELINE.json north_star): tile assignments / sorted keys / per-tile ranges bit-exact,
images within 1e-4 absolute, gradients within 1e-3 relative (norm-relative floor).
"""
import numpy as np
import pytest

from paper_2404_03202_b200 import native, scenes

from parity import IMAGE_ATOL, assert_grads_close, compare_projections, compare_tiles

pytestmark = pytest.mark.gpu


def _scene(kind, n, seed=1):
    return scenes.synthetic_cloud(n, seed=seed, variant=kind)


CASES = [
    # (name, cloud factory, pose, W, H)
    ("c1_uniform", lambda: _scene("uniform", 10_000, 1), scenes.identity_pose(), 512, 256),
    ("pole_small", lambda: _scene("pole", 3_000, 3), scenes.identity_pose(), 256, 128),
    ("seam_small", lambda: _scene("seam", 3_000, 4), scenes.identity_pose(), 256, 128),
    ("random_pose", lambda: _scene("uniform", 5_000, 5), scenes.random_pose(np.random.default_rng(7)), 384, 192),
    ("odd_size", lambda: _scene("uniform", 2_000, 6), scenes.identity_pose(), 200, 100),
]


@pytest.mark.parametrize("name,make,pose,W,H", CASES, ids=[c[0] for c in CASES])
def test_forward_parity(name, make, pose, W, H, oracle_port):
    cloud = make()
    ctx = native.Context(cloud)
    fr = ctx.render(pose, W, H)
    of = oracle_port.render(cloud, pose, W, H)

    proj = compare_projections(fr, of, cloud.n)
    # FP64 on both sides; CUDA atan2/asin/exp differ from glibc by <= 2 ulp, which the
    # (s + 1) * W / 2 map turns into ~1e-13 px near the seam/poles.
    assert proj["p_abs"] < 1e-9, proj
    assert proj["conic_rel"] < 1e-9, proj
    assert proj["opacity_rel"] < 1e-14, proj
    assert proj["color_abs"] < 1e-6, proj
    assert proj["touched_mismatch"] == 0, proj

    nbad, first = compare_tiles(fr, of)
    assert nbad == 0, f"{nbad} tile lists differ (first {first})"

    rgb, T, con, last = fr.pixels()
    img = fr.image()
    err = np.max(np.abs(img - of.rgb))
    assert err <= IMAGE_ATOL, err
    assert np.array_equal(last, of.last_contrib), int(np.sum(last != of.last_contrib))
    assert np.array_equal(con, of.contributors), int(np.sum(con != of.contributors))
    assert np.max(np.abs(T - of.T)) < 1e-5


@pytest.mark.parametrize("name,make,pose,W,H", CASES[:4], ids=[c[0] for c in CASES[:4]])
def test_backward_parity(name, make, pose, W, H, oracle_port):
    cloud = make()
    rng = np.random.default_rng(11)
    d_image = rng.uniform(-1.0, 1.0, size=(H, W, 3)) / (W * H)
    ctx = native.Context(cloud)
    fr = ctx.render(pose, W, H)
    ctx.backward(fr, d_image)
    g = ctx.gradients()
    of = oracle_port.render(cloud, pose, W, H, keep_handle=True)
    go = oracle_port.backward(of, d_image, cloud, pose)
    oracle_port.free(of)
    assert_grads_close(g, go)
    assert np.array_equal(g["screen_hits"], go.screen_hits)
    ds_scale = np.max(np.abs(go.d_screen))
    assert np.max(np.abs(g["d_screen"] - go.d_screen)) <= 1e-3 * ds_scale + 1e-12


def test_adam_parity(oracle_port):
    """adam_step over the GPU's own FP32 gradients vs the oracle fed the same gradients."""
    import pyoracle
    cloud = _scene("uniform", 4_000, 9)
    W, H, pose = 256, 128, scenes.identity_pose()
    ctx = native.Context(cloud)
    ref = cloud.copy()
    st = pyoracle.AdamState.zeros(cloud.n, cloud.basis_count)
    cfg = pyoracle.AdamConfig(iterations=100)
    ncfg = native.Config(iterations=100)
    rng = np.random.default_rng(3)
    for it in range(1, 11):
        fr = ctx.render(pose, W, H)
        d_image = rng.uniform(-1.0, 1.0, size=(H, W, 3)) / (W * H)
        ctx.backward(fr, d_image)
        g = ctx.gradients()
        go = pyoracle.Grads(g["d_position"], g["d_sh"], g["d_rotation"], g["d_log_scale"], g["d_opacity_logit"],
                            g["d_screen"], np.zeros(cloud.n), np.zeros(cloud.n, dtype=np.int64))
        ctx.adam_step(ncfg, 1.5, it)
        oracle_port.adam_step(ref, go, st, cfg, 1.5, it)
        fr.free()
        got = ctx.download()
        # oracle keeps FP64 params; the device keeps FP32 planes -> compare within FP32 rounding of
        # the accumulated update (lr-scaled)
        for name, lr in (("positions", 1.6e-4 * 1.5), ("sh", 2.5e-3), ("rotations", 1e-3), ("log_scales", 5e-3),
                         ("opacity_logits", 5e-2)):
            a, b = getattr(got, name), getattr(ref, name)
            tol = 1e-6 * np.abs(b) + 1e-3 * lr * it
            assert np.all(np.abs(a - b) <= tol + 1e-7), (name, it, float(np.max(np.abs(a - b))))
        # resync the oracle to the device's FP32 parameters so FP32 rounding does not compound
        ref = got.copy()


def test_tiled_matches_bruteforce_compact(oracle_port):
    """test_rasterizer.cpp:171-185 through the GPU: 50 compact scenes, |tiled - brute| < 1e-5."""
    rng = np.random.default_rng(43)
    worst = 0.0
    for scene in range(50):
        cloud = scenes.random_cloud(rng, count=20 + scene % 80, min_opacity=0.05, max_opacity=0.3)
        pose = scenes.random_pose(rng)
        ctx = native.Context(cloud)
        img = ctx.render(pose, 128, 64).image()
        ref = oracle_port.render(cloud, pose, 128, 64, brute_force=True)
        worst = max(worst, float(np.max(np.abs(img - ref.rgb))))
    assert worst < 1e-5, worst


def test_osplat_render_c_abi_matches_frame(oracle_port):
    cloud = _scene("uniform", 3_000, 12)
    pose = scenes.random_pose(np.random.default_rng(1))
    hc = native.HostCloud.from_cloud(cloud)
    img = native.osplat_render(hc, pose, 256, 128)
    of = oracle_port.render(cloud, pose, 256, 128)
    assert img.shape == (128, 256, 3)
    assert np.max(np.abs(img - of.rgb)) <= IMAGE_ATOL


def test_osplat_render_banded_copy_and_rerender(oracle_port):
    """osplat_render blends in bands of tile rows and copies each band to the host image while the
    next blends (Engine::render_hwc); an odd-sized image (partial last tile row) and a frame whose
    instances outgrow the pooled buffer (re-rendered on validation, then copied again) must both
    equal the oracle."""
    cloud = _scene("uniform", 4_000, 15)
    hc = native.HostCloud.from_cloud(cloud)
    pose = scenes.random_pose(np.random.default_rng(3))
    small = native.osplat_render(hc, pose, 64, 32)  # sizes the cloud's pooled frame small
    of_small = oracle_port.render(cloud, pose, 64, 32)
    assert np.max(np.abs(small - of_small.rgb)) <= IMAGE_ATOL
    for W, H in ((520, 250), (512, 256)):  # the first outgrows the pool and is re-rendered
        img = native.osplat_render(hc, pose, W, H)
        of = oracle_port.render(cloud, pose, W, H)
        assert img.shape == (H, W, 3)
        assert np.max(np.abs(img - of.rgb)) <= IMAGE_ATOL, (W, H)


def test_empty_and_culled_clouds():
    empty = scenes.synthetic_cloud(0, seed=1)
    ctx = native.Context(empty)
    img = ctx.render(scenes.identity_pose(), 128, 64, background=(0.2, 0.3, 0.4)).image()
    assert np.allclose(img[..., 0], 0.2) and np.allclose(img[..., 2], 0.4)
    faint = scenes.synthetic_cloud(100, seed=2)
    faint.opacity_logits[:] = -10.0  # sigmoid < 1/255 -> every Gaussian culled
    ctx = native.Context(faint)
    fr = ctx.render(scenes.identity_pose(), 128, 64)
    assert np.all(fr.image() == 0.0)
    assert fr.tiles()[3].size == 0


@pytest.mark.parametrize("legacy", [False, True])
def test_context_adopts_caller_stream(legacy):
    """Kernels run on the caller's stream (torch events on it bracket them; NCCL ordering)."""
    import torch
    s = torch.cuda.default_stream() if legacy else torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = native.Context(_scene("uniform", 50_000, 2), stream=s.cuda_stream)
        ctx.profile(timing=True)
        ctx.render(scenes.identity_pose(), 1024, 512).free()  # warm
        ctx.profile_read(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            ctx.render(scenes.identity_pose(), 1024, 512).free()
        e1.record(s)
        torch.cuda.synchronize()
        kern = sum(v[0] for v in ctx.profile_read().values())
        assert kern > 0.0
        assert e0.elapsed_time(e1) >= 0.9 * kern, (e0.elapsed_time(e1), kern)


def test_accumulate_and_logical_zero():
    """backward(accumulate) sums views; a consuming Adam step / zero_grad makes the next backward
    start from zero (the planes are overwritten, never read)."""
    cloud = _scene("uniform", 4000, 13)
    W, H = 256, 128
    pa, pb = scenes.identity_pose(), scenes.random_pose(np.random.default_rng(3))
    rng = np.random.default_rng(5)
    da = rng.uniform(-1, 1, size=(H, W, 3)) / (W * H)
    db = rng.uniform(-1, 1, size=(H, W, 3)) / (W * H)
    ctx = native.Context(cloud)
    fa, fb = ctx.render(pa, W, H), ctx.render(pb, W, H)
    ctx.backward(fa, da)
    ga = ctx.gradients()
    ctx.backward(fb, db)
    gb = ctx.gradients()
    ctx.zero_grad()
    ctx.backward(fa, da, accumulate=True)
    ctx.backward(fb, db, accumulate=True)
    gab = ctx.gradients()
    for k in ("d_position", "d_sh", "d_rotation", "d_log_scale", "d_opacity_logit"):
        ref = ga[k] + gb[k]
        # each backward is recomputed: K4a's FP32 atomics reorder its sums run to run
        assert np.allclose(gab[k], ref, rtol=1e-4, atol=1e-6 * np.max(np.abs(ref))), k
    ctx.adam_step(native.Config(), 1.0, 1, zero_grad=True)
    fa.free()
    fa = ctx.render(pa, W, H)
    ctx.backward(fa, da, accumulate=True)
    g1 = ctx.gradients()
    ctx.backward(fa, da)  # reference overwrite semantics
    g2 = ctx.gradients()
    for k in ("d_position", "d_sh", "d_rotation", "d_log_scale", "d_opacity_logit"):
        # K4a's FP32 atomics make the summation order run-dependent
        assert np.allclose(g1[k], g2[k], rtol=1e-4, atol=1e-6 * np.max(np.abs(g2[k]))), k


def test_backward_with_background(oracle_port):
    """The background term of d_alpha (gradients.cpp:142) and of the pixel colour."""
    cloud = _scene("uniform", 3000, 17)
    pose = scenes.random_pose(np.random.default_rng(19))
    W, H, bg = 256, 128, (0.3, 0.6, 0.9)
    d_image = np.random.default_rng(23).uniform(-1.0, 1.0, size=(H, W, 3)) / (W * H)
    ctx = native.Context(cloud)
    fr = ctx.render(pose, W, H, background=bg)
    of = oracle_port.render(cloud, pose, W, H, bg, keep_handle=True)
    assert np.max(np.abs(fr.image() - of.rgb)) <= IMAGE_ATOL
    ctx.backward(fr, d_image)
    g = ctx.gradients()
    go = oracle_port.backward(of, d_image, cloud, pose)
    oracle_port.free(of)
    assert_grads_close(g, go)


@pytest.mark.parametrize("active", [0, 1, 2])
def test_active_sh_degree(active, oracle_port):
    """Renders and gradients with fewer active SH bands than stored (sh_warmup)."""
    cloud = _scene("uniform", 2000, 29)
    cloud.active_sh_degree = active
    pose = scenes.identity_pose()
    W, H = 192, 96
    d_image = np.random.default_rng(31).uniform(-1.0, 1.0, size=(H, W, 3)) / (W * H)
    ctx = native.Context(cloud)
    fr = ctx.render(pose, W, H)
    of = oracle_port.render(cloud, pose, W, H, keep_handle=True)
    assert np.max(np.abs(fr.image() - of.rgb)) <= IMAGE_ATOL
    ctx.backward(fr, d_image)
    g = ctx.gradients()
    go = oracle_port.backward(of, d_image, cloud, pose)
    oracle_port.free(of)
    bc_active = (active + 1) ** 2
    assert np.all(g["d_sh"][:, bc_active:, :] == 0.0)
    assert_grads_close(g, go)


def test_instance_buffer_growth_rerenders_exactly(oracle_port):
    """Frames are enqueued without a host sync; a frame whose instances outgrow the pooled buffer
    is re-rendered on first use (Engine::validate) and must still equal the oracle."""
    cloud = scenes.synthetic_cloud(3000, seed=13)
    ctx = native.Context(cloud)
    ctx.render(scenes.identity_pose(), 64, 32).free()  # sizes the pooled frame for ~1/16 the instances
    pose = scenes.random_pose(np.random.default_rng(4))
    fr = ctx.render(pose, 512, 256)
    of = oracle_port.render(cloud, pose, 512, 256)
    nbad, first = compare_tiles(fr, of)
    assert nbad == 0, (nbad, first)
    assert np.max(np.abs(fr.image() - of.rgb)) <= IMAGE_ATOL
    fr.free()


def test_equal_depth_runs_fall_back_to_the_exact_sort(oracle_port):
    """More than 32 Gaussians at bit-identical depth defeat the FP32-key fast path; the frame is
    re-rendered with the 64-bit depth sort and the (depth, id) order stays exact."""
    cloud = scenes.synthetic_cloud(2000, seed=14)
    # 64 copies of one Gaussian's position (identical t_r), spread colours
    cloud.positions[100:164] = cloud.positions[100]
    cloud.sh[100:164, 0, :] = np.linspace(-0.4, 0.4, 64)[:, None]
    ctx = native.Context(cloud)
    pose = scenes.identity_pose()
    fr = ctx.render(pose, 256, 128)
    of = oracle_port.render(cloud, pose, 256, 128)
    nbad, first = compare_tiles(fr, of)
    assert nbad == 0, (nbad, first)
    assert np.max(np.abs(fr.image() - of.rgb)) <= IMAGE_ATOL


def test_depth_runs_straddling_emission_blocks(oracle_port):
    """Runs of FP32-equal depth keys: groups of 2..40 Gaussians moved off one position along a
    tangent by permuted multiples of 5e-5 (FP64-distinct depths that round to one FP32 value, in
    an order unrelated to their ids) put ~98 % of the depth ranks in 1,331 runs of up to 21, four
    of them straddling the 2048-rank blocks of the emission scan: every member places itself at its
    exact (FP64 depth, id) position inside its run (k_touch_sums) and the tile lists stay the
    oracle's."""
    rng = np.random.default_rng(21)
    cloud = scenes.synthetic_cloud(9000, seed=21)
    P = cloud.positions.copy()
    i = 0
    while i < 9000:
        L = int(rng.integers(2, 41))
        idx = np.arange(i, min(i + L, 9000))
        e = np.cross(P[i], [0.3, 1.0, 0.2])
        e /= np.linalg.norm(e)
        P[idx] = P[i] + (5e-5 * rng.permutation(len(idx)))[:, None] * e
        i += L
    cloud.positions = P
    cloud = cloud.rounded()  # the device holds FP32 parameters: the oracle sees the same values
    ctx = native.Context(cloud)
    pose = scenes.identity_pose()
    fr = ctx.render(pose, 384, 192)
    of = oracle_port.render(cloud, pose, 384, 192)
    nbad, first = compare_tiles(fr, of)
    assert nbad == 0, (nbad, first)
    assert np.max(np.abs(fr.image() - of.rgb)) <= IMAGE_ATOL
    fr.free()


def test_adam_shards_equal_the_full_step():
    """osplat_gpu_adam_step_range over the shards of a data-parallel world == the full fused Adam,
    bit for bit (the sharded optimizer's update is elementwise)."""
    import torch

    from paper_2404_03202_b200 import dp
    cloud = scenes.synthetic_cloud(3000, seed=15)
    rng = np.random.default_rng(2)
    cfg = native.Config(iterations=100)
    d = rng.uniform(-1, 1, size=(64, 128, 3)) / (64 * 128)
    world = 4
    ctxs = [native.Context(cloud) for _ in range(world + 1)]
    for c in ctxs:
        fr = c.render(scenes.identity_pose(), 128, 64)
        c.backward(fr, d)
        fr.free()
    grads = lambda c: torch.as_tensor(dp._CudaArray(c.view().grads, c.view().planes * c.view().stride),
                                      device="cuda")
    for c in ctxs[1:]:  # K4a's FP32 atomics make gradients order-dependent: give all the same ones
        grads(c).copy_(grads(ctxs[0]))
    torch.cuda.synchronize()
    ctxs[0].adam_step(cfg, 1.0, 1)
    flat = lambda c: torch.as_tensor(dp._CudaArray(c.view().params, c.view().planes * c.view().stride),
                                     device="cuda").cpu().numpy()
    full = flat(ctxs[0])
    for r in range(world):
        c = ctxs[1 + r]
        b, n = dp.shard_range(full.size, r, world)
        before = flat(c)
        c.adam_step(cfg, 1.0, 1, begin=b, count=n)
        after = flat(c)
        assert np.array_equal(after[b:b + n], full[b:b + n]), r
        outside = np.ones(full.size, dtype=bool)
        outside[b:b + n] = False
        assert np.array_equal(after[outside], before[outside]), r
