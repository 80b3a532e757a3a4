"""GPU: the CUDA backward against central finite differences of the reference's FP64 forward model
(every gradient path — position through the mean and the covariance, SH,
quaternion, log-scale, opacity — matches central differences within 1e-3 relative).

For small random scenes (the reference's test scene, tests/test_utils.hpp:52-90) and a linear loss
L = sum w * C with fixed random w (so dL/dC = w exactly), the GPU gradient of every parameter is
compared with the validated central difference (test_utils.hpp:97-112: the estimates at h and h/2
must agree, else the step shrinks; a blend threshold inside the stencil makes it meaningless) of
L evaluated by the FP64 oracle render. This pins the backward to the derivative of the forward
model itself, independently of the reference's own backward()."""
import numpy as np
import pytest

from paper_2404_03202_b200 import native, scenes

pytestmark = pytest.mark.gpu

W, H = 64, 32
GROUPS = [("positions", "d_position", 1e-4), ("sh", "d_sh", 1e-3), ("rotations", "d_rotation", 1e-4),
          ("log_scales", "d_log_scale", 1e-4), ("opacity_logits", "d_opacity_logit", 1e-3)]


def _validated_fd(f, x, h0):
    h = h0
    for _ in range(3):
        d1 = (f(x + h) - f(x - h)) / (2.0 * h)
        d2 = (f(x + h / 2) - f(x - h / 2)) / h
        scale = max(abs(d1), abs(d2), 1e-8)
        if abs(d1 - d2) <= 1e-4 * scale:
            return d2, True
        h /= 16.0
    return 0.0, False


@pytest.mark.parametrize("seed", range(6))
def test_backward_matches_finite_differences(seed, oracle_port):
    rng = np.random.default_rng(1000 + seed)
    cloud = scenes.random_cloud(rng, count=12 + 3 * seed)
    pose = scenes.random_pose(rng)
    w = rng.uniform(-1.0, 1.0, size=(H, W, 3))
    ctx = native.Context(cloud)
    fr = ctx.render(pose, W, H)
    ctx.backward(fr, w)
    g = ctx.gradients()
    fr.free()

    checked = 0
    for field, gkey, h0 in GROUPS:
        base = getattr(cloud, field)
        grad = np.asarray(g[gkey]).reshape(base.shape)
        flat = base.reshape(-1)
        fd = np.zeros(flat.size)
        ok = np.zeros(flat.size, dtype=bool)
        for i in range(flat.size):
            def f(x, i=i):
                c = cloud.copy()
                arr = getattr(c, field).reshape(-1)
                arr[i] = x
                setattr(c, field, arr.reshape(base.shape))
                return float(np.sum(w * oracle_port.render(c, pose, W, H).rgb))
            fd[i], ok[i] = _validated_fd(f, flat[i], h0 * max(1.0, abs(flat[i])))
        gv = grad.reshape(-1)
        scale = max(np.max(np.abs(fd[ok])), 1e-12) if ok.any() else 1.0
        tol = np.maximum(1e-3 * np.maximum(np.abs(gv), np.abs(fd)), 1e-4 * scale)
        bad = ok & (np.abs(gv - fd) > tol)
        assert not bad.any(), (field, np.nonzero(bad)[0][:5], gv[bad][:5], fd[bad][:5])
        checked += int(ok.sum())
    assert checked > 0.9 * sum(getattr(cloud, f).size for f, _, _ in GROUPS)
