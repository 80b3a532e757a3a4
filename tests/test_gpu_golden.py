"""GPU: the CUDA path against the committed golden fixtures (tests/golden/*.npz), produced by the
REFERENCE's own sources (oracle/_ref) with tests/golden/make_golden.py. These pin the GPU path
directly on a box without /root/reference, independently of the C restatement:

* projections (visible set, centre, conic, radius, depth, colour) of K1;
* tile lists (K2) bit-exact; image within 1e-4, T, contributors / last_contrib (K3);
* GradientBuffer of the fixture's d_image (K4a/K4b), every entry within 1e-3 relative;
* parameters after 1 and 10 fused Adam steps (K5) on the fixture's gradients.
"""
import glob
import os

import numpy as np
import pytest

from paper_2404_03202_b200 import native, scenes

from parity import IMAGE_ATOL, assert_grads_close

pytestmark = pytest.mark.gpu

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def _load(path):
    d = np.load(path)
    cloud = scenes.Cloud(d["positions"], d["sh"], d["rotations"], d["log_scales"], d["opacity_logits"],
                         int(d["sh_degree"]), int(d["active_sh_degree"]))
    return d, cloud


class _G:
    def __init__(self, d):
        for k in ("d_position", "d_sh", "d_rotation", "d_log_scale", "d_opacity_logit", "d_screen"):
            setattr(self, k, d["g_" + k])


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_render_and_backward_match_golden(path):
    d, cloud = _load(path)
    W, H, pose, bg = int(d["width"]), int(d["height"]), d["pose"], tuple(d["background"])
    ctx = native.Context(cloud)
    fr = ctx.render(pose, W, H, background=bg)
    pr = fr.projections()
    gid = d["f_gid"]
    vis = np.zeros(cloud.n, dtype=bool)
    vis[gid] = True
    assert np.array_equal(pr["visible"], vis)
    assert np.max(np.abs(pr["p"][gid] - d["f_p"]), initial=0.0) < 1e-9
    assert np.max(np.abs(pr["conic"][gid] - d["f_conic"]) / np.abs(d["f_conic"]).clip(1e-300), initial=0.0) < 1e-9
    assert np.max(np.abs(pr["color"][gid] - d["f_color"]), initial=0.0) < 1e-6
    # tile lists: the fixture stores projection indices per tile (TileGrid); map to Gaussian ids
    tx, ty, ranges, ids = fr.tiles()
    offs, items = d["f_offsets"], d["f_items"]
    assert tx * ty + 1 == offs.size
    for t in range(tx * ty):
        assert np.array_equal(ids[ranges[t, 0]:ranges[t, 1]], gid[items[offs[t]:offs[t + 1]]]), t
    rgb, T, con, last = fr.pixels()
    assert np.max(np.abs(fr.image() - d["f_rgb"])) <= IMAGE_ATOL
    assert np.max(np.abs(T - d["f_T"])) < 1e-5
    assert np.array_equal(con, d["f_contributors"]) and np.array_equal(last, d["f_last"])
    ctx.backward(fr, d["d_image"])
    g = ctx.gradients()
    fr.free()
    assert_grads_close(g, _G(d))
    ds = np.max(np.abs(d["g_d_screen"]))
    assert np.max(np.abs(g["d_screen"] - d["g_d_screen"])) <= 1e-3 * ds + 1e-15


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_adam_matches_golden(path):
    """adam_step (trainer.cpp:143-178) x 10 on the fixture's reference gradients (uploaded into
    the device gradient planes), extent 1.25, iterations 30."""
    import torch

    from paper_2404_03202_b200 import dp
    d, cloud = _load(path)
    ctx = native.Context(cloud)
    v = ctx.view()
    n, bc, stride = cloud.n, cloud.basis_count, v.stride
    planes = np.zeros((v.planes, stride), dtype=np.float32)
    planes[0:3, :n] = d["g_d_position"].T
    for b in range(bc):
        for c in range(3):
            planes[3 + 3 * b + c, :n] = d["g_d_sh"][:, b, c]
    planes[3 + 3 * bc:7 + 3 * bc, :n] = d["g_d_rotation"].T
    planes[7 + 3 * bc:10 + 3 * bc, :n] = d["g_d_log_scale"].T
    planes[10 + 3 * bc, :n] = d["g_d_opacity_logit"]
    grads = torch.as_tensor(dp._CudaArray(v.grads, v.planes * stride), device="cuda")
    grads.copy_(torch.from_numpy(planes.ravel()))
    torch.cuda.synchronize()
    cfg = native.Config(iterations=int(d["adam_iterations"]))
    extent = float(d["extent"])
    for it in range(1, 11):
        ctx.adam_step(cfg, extent, it, zero_grad=False)
        if it in (1, 10):
            got = ctx.download()
            for name, lr in (("positions", 1.6e-4 * extent), ("sh", 2.5e-3), ("rotations", 1e-3),
                             ("log_scales", 5e-3), ("opacity_logits", 5e-2)):
                a, b = getattr(got, name), d[f"adam{it}_{name}"]
                # FP32 parameters / moments vs the reference's doubles: the FP32 rounding of each
                # parameter plus <= 1e-3 of the accumulated (lr-bounded) update
                tol = 2e-7 * np.abs(b) + 1e-3 * lr * it + 1e-12
                assert np.all(np.abs(a - b) <= tol), (name, it, float(np.max(np.abs(a - b) - tol)))
