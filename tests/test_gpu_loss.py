"""GPU parity of the device loss (L1 + SSIM with gradient, bottom-row mask) against the oracle's
loss() (trainer.cpp:25-71, metrics.cpp:81-153) on identical inputs (our FP32 render, FP32 target)."""
import numpy as np
import pytest

from paper_2404_03202_b200 import native, scenes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("lam,mask,W,H", [(0.0, 0.0, 256, 128), (0.2, 0.0, 256, 128), (0.2, 0.1, 200, 100),
                                           (1.0, 0.25, 96, 48)])
def test_loss_matches_oracle(lam, mask, W, H, oracle_port):
    import torch
    cloud = scenes.synthetic_cloud(3000, seed=3)
    target = scenes.synthetic_cloud(3000, seed=4)
    pose = scenes.identity_pose()
    ctx = native.Context(cloud)
    tctx = native.Context(target)
    fr = ctx.render(pose, W, H)
    rgb32, _, _, _ = fr.pixels()
    gt32, _, _, _ = tctx.render(pose, W, H).pixels()
    gt_dev = torch.from_numpy(np.ascontiguousarray(gt32.transpose(2, 0, 1))).cuda()
    torch.cuda.synchronize()
    value, dptr = ctx.loss(fr, gt_dev.data_ptr(), lam, mask)
    d = torch.empty(3 * W * H, dtype=torch.float32, device="cuda")
    d.copy_(torch.as_tensor(_Dev(dptr, 3 * W * H), device="cuda"))
    d_gpu = d.cpu().numpy().reshape(3, H, W).transpose(1, 2, 0)
    v_or, d_or = oracle_port.loss(rgb32.astype(np.float64), gt32.astype(np.float64), lam, mask)
    assert abs(value - v_or) <= 1e-5 * max(abs(v_or), 1e-6), (value, v_or)
    scale = np.max(np.abs(d_or))
    assert np.max(np.abs(d_gpu - d_or)) <= 1e-4 * scale, float(np.max(np.abs(d_gpu - d_or)) / scale)
    keep = H - int(np.floor(mask * H))
    assert np.all(d_gpu[keep:] == 0.0)


class _Dev:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "strides": None}


def test_train_view_async_matches_sync():
    """osplat_gpu_train_view_async enqueues the step without waiting; its loss sums (pinned host)
    give the same loss as the synchronous osplat_gpu_train_view, and the accumulated gradients agree."""
    import torch
    W, H = 256, 128
    cloud = scenes.synthetic_cloud(4000, seed=5)
    gt32, _, _, _ = native.Context(scenes.synthetic_cloud(4000, seed=6)).render(scenes.identity_pose(), W, H).pixels()
    gt = np.ascontiguousarray(gt32.transpose(2, 0, 1))
    pose = scenes.ring_poses(4, seed=2)[1]
    a, b = native.Context(cloud), native.Context(cloud)
    la = a.train_view(pose, W, H, gt, gt_on_device=False, lambda_ssim=0.2, mask=0.1)
    sums = torch.zeros(4, dtype=torch.float64, pin_memory=True)
    b.train_view_async(pose, W, H, gt, gt_on_device=False, sums_ptr=sums.data_ptr(), lambda_ssim=0.2, mask=0.1)
    b.synchronize()
    lb = native.loss_value(sums.numpy(), 0.2, W, H, 0.1)
    assert abs(la - lb) <= 1e-12 * abs(la), (la, lb)
    ga, gb = a.gradients(), b.gradients()
    for k in ("d_position", "d_sh", "d_opacity_logit"):
        scale = np.max(np.abs(ga[k]))
        assert np.max(np.abs(ga[k] - gb[k])) <= 1e-4 * scale, k
