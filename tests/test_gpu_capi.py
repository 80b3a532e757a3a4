"""GPU: the reference C ABI entry points beyond render — osplat_metrics (capi.h:90-92) against the
reference's psnr / ssim (metrics.cpp:64-79), and concurrent osplat_render calls on one read-shared
cloud."""
import threading

import numpy as np
import pytest

from paper_2404_03202_b200 import native, scenes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("H,W", [(5, 7), (64, 128), (512, 1024)])
def test_osplat_metrics_matches_reference(H, W, oracle_ref):
    rng = np.random.default_rng(H * 31 + W)
    a = rng.uniform(0, 1, (H, W, 3))
    b = np.clip(a + rng.normal(0, 0.05, a.shape), 0, 1)
    ps, ss = native.osplat_metrics(a, b)
    pr, sr = oracle_ref.metrics(a, b)
    # FP64 on both sides; only the summation order of the device reductions differs
    assert abs(ps - pr) <= 1e-9 * abs(pr), (ps, pr)
    assert abs(ss - sr) <= 1e-12, (ss, sr)
    assert native.osplat_metrics(a, a) == (99.0, 1.0)  # kPsnrCap for zero MSE


def test_osplat_metrics_of_renders(oracle_ref):
    """PSNR / SSIM between two GPU renders (osplat_render -> osplat_image), as the reference's
    training hook computes them (capi.cpp:212-214)."""
    cloud = scenes.synthetic_cloud(20_000, seed=3)
    hc = native.HostCloud.from_cloud(cloud)
    p0, p1 = scenes.ring_poses(2, seed=4)
    a = native.osplat_render(hc, p0, 512, 256)
    b = native.osplat_render(hc, p1, 512, 256)
    ps, ss = native.osplat_metrics(a, b)
    pr, sr = oracle_ref.metrics(a, b)
    assert abs(ps - pr) <= 1e-9 * abs(pr) and abs(ss - sr) <= 1e-12


def test_osplat_metrics_size_mismatch():
    with pytest.raises(native.OsplatError) as e:
        native.osplat_metrics(np.zeros((4, 6, 3)), np.zeros((4, 7, 3)))
    assert e.value.status == native.VALIDATION
    assert e.value.message.startswith("DimensionMismatch: ")


def test_concurrent_osplat_render_on_one_cloud():
    """Four host threads render one const cloud at once (the reference's osplat_render is a pure
    function of a read-shared cloud): every image equals the single-threaded render."""
    cloud = scenes.synthetic_cloud(50_000, seed=8)
    hc = native.HostCloud.from_cloud(cloud)
    poses = scenes.ring_poses(8, seed=9)
    W, H = 512, 256
    expect = [native.osplat_render(hc, p, W, H) for p in poses]
    hc2 = native.HostCloud.from_cloud(cloud)  # fresh cloud: its device copy is created under the race
    errors, results = [], {}

    def worker(t):
        try:
            for k in range(len(poses)):
                j = (k + 2 * t) % len(poses)
                results[(t, k)] = (j, native.osplat_render(hc2, poses[j], W, H))
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    assert len(results) == 4 * len(poses)
    for j, img in results.values():
        assert np.array_equal(img, expect[j])


@pytest.mark.parametrize("crop", [False, True], ids=["omnidirectional", "perspective_crop"])
def test_osplat_gpu_eval_matches_reference_metrics(crop, oracle_ref):
    """osplat_gpu_eval (osplat_eval / run_eval, eval.cpp:63-116): per-view PSNR / SSIM of the GPU
    render against each target equal the reference's psnr / ssim of the same images (on the
    panorama, or averaged over its 6 cube-face crops made by the reference's perspective_crop)."""
    cloud = scenes.synthetic_cloud(30_000, seed=5)
    target = scenes.synthetic_cloud(30_000, seed=6)
    poses = scenes.ring_poses(6, seed=7)
    W, H = 256, 128
    t = native.Context(target)
    images = []
    for p in poses:
        fr = t.render(p, W, H)
        images.append(fr.image())
        fr.free()
    is_test = [k % 2 == 0 for k in range(len(poses))]
    ctx = native.Context(cloud)
    rep = ctx.eval(poses, images, is_test, split="test", perspective_crop=crop)
    assert rep["mode"] == ("perspective-crop" if crop else "omnidirectional")
    assert [v[0] for v in rep["views"]] == [0, 2, 4]
    assert rep["fps"] > 0 and abs(rep["fps"] * rep["seconds_per_frame"] - 1.0) < 1e-9
    for fi, ps, ss in rep["views"]:
        fr = ctx.render(poses[fi], W, H)
        img = fr.image()
        fr.free()
        if crop:
            rc, gc = oracle_ref.cube_crops(img, H // 2), oracle_ref.cube_crops(images[fi], H // 2)
            ms = [oracle_ref.metrics(rc[k], gc[k]) for k in range(6)]
            pr, sr = np.mean([m[0] for m in ms]), np.mean([m[1] for m in ms])
        else:
            pr, sr = oracle_ref.metrics(img, images[fi])
        assert abs(ps - pr) <= 1e-8 * abs(pr) and abs(ss - sr) <= 1e-10, (fi, ps, pr, ss, sr)
    assert abs(rep["mean_psnr"] - np.mean([v[1] for v in rep["views"]])) < 1e-9
    assert len(ctx.eval(poses, images, is_test, split="all")["views"]) == 6
    with pytest.raises(native.OsplatError) as e:
        ctx.eval(poses, images, None, split="test")
    assert e.value.status == native.VALIDATION and e.value.message.startswith("EmptySplit: ")
    with pytest.raises(native.OsplatError) as e:
        ctx.eval(poses, images, is_test, split="bogus")
    assert e.value.status == native.INVALID_ARGUMENT
