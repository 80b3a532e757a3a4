"""GPU: the fused single-view training step (osplat_gpu_backward_step / osplat_gpu_train_step_async)
— backward with the SH gradients consumed by Adam in place — equals backward(overwrite) +
adam_step (trainer.cpp:363 + 381) bit for bit: parameters and Adam moments, every SH degree, culled
Gaussians included (deterministic backward on both, so both sides see the same gradients)."""
import numpy as np
import pytest

from paper_2404_03202_b200 import dp, native, scenes

pytestmark = pytest.mark.gpu

FIELDS = ("positions", "sh", "rotations", "log_scales", "opacity_logits")


def _moments(ctx):
    import torch
    v = ctx.view()
    n = v.planes * v.stride
    m = torch.as_tensor(dp._CudaArray(v.adam_m, n), device="cuda").cpu().numpy()
    s = torch.as_tensor(dp._CudaArray(v.adam_v, n), device="cuda").cpu().numpy()
    return m, s


def _target(cloud_seed, n, poses, W, H):
    import torch
    t = native.Context(scenes.synthetic_cloud(n, seed=cloud_seed))
    out = []
    for p in poses:
        fr = t.render(p, W, H)
        g = torch.empty(3 * W * H, dtype=torch.float32, device="cuda")
        g.copy_(torch.as_tensor(dp._CudaArray(fr.device().rgb, 3 * W * H), device="cuda"))
        out.append(g)
        fr.free()
    return out


@pytest.mark.parametrize("active", [0, 1, 3])
def test_backward_step_equals_backward_plus_adam(active):
    import torch
    W, H = 384, 192
    cloud = scenes.synthetic_cloud(20_000, seed=61)
    cloud.opacity_logits[::50] = -9.0  # culled (opacity < 1/255): Adam still moves them with g = 0
    cloud.active_sh_degree = active
    poses = scenes.ring_poses(3, seed=62)
    gts = _target(63, 20_000, poses, W, H)
    cfg = native.Config(iterations=50)
    res = []
    for fused in (False, True):
        ctx = native.Context(cloud)
        ctx.set_deterministic(True)
        for it in range(1, 4):
            fr = ctx.render(poses[it - 1], W, H)
            _, dimg = ctx.loss(fr, gts[it - 1].data_ptr(), 0.2, 0.0, want_value=False)
            if fused:
                ctx.backward_step(fr, dimg, cfg, 1.3, it)
            else:
                ctx.backward_device(fr, dimg, accumulate=False)
                ctx.adam_step(cfg, 1.3, it, zero_grad=True)
            fr.free()
        torch.cuda.synchronize()
        res.append((ctx.download(), _moments(ctx), ctx.view().adam_step))
        ctx.free()
    (a, (ma, va), sa), (b, (mb, vb), sb) = res
    assert sa == sb == 3
    for f in FIELDS:
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(ma, mb) and np.array_equal(va, vb)


def test_train_step_async_equals_train_view_plus_adam():
    """The pipelined C-ABI step (host target in, loss sums out) with the fused backward + Adam."""
    import torch
    W, H = 256, 128
    cloud = scenes.synthetic_cloud(10_000, seed=71)
    poses = scenes.ring_poses(4, seed=72)
    gts = [g.cpu().numpy() for g in _target(73, 10_000, poses, W, H)]
    cfg = native.Config(iterations=40)
    res = []
    for fused in (False, True):
        ctx = native.Context(cloud)
        ctx.set_deterministic(True)
        sums = torch.zeros((4, 4), dtype=torch.float64, pin_memory=True)
        for it in range(1, 5):
            if fused:
                ctx.train_step_async(poses[it - 1], W, H, gts[it - 1], False, sums[it - 1].data_ptr(), cfg, 1.0, it)
            else:
                ctx.train_view_async(poses[it - 1], W, H, gts[it - 1], False, sums[it - 1].data_ptr())
                ctx.adam_step(cfg, 1.0, it, zero_grad=True)
        ctx.synchronize()
        res.append((ctx.download(), sums.numpy().copy()))
        ctx.free()
    (a, sa), (b, sb) = res
    for f in FIELDS:
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(sa[:, 0], sb[:, 0])  # L1 sums of the same renders
