"""Generate the golden fixtures from the REFERENCE sources (oracle/_ref/libref_oracle.so, built from
/root/reference by oracle/Makefile). Run here, where the reference tree exists:

    make -C oracle && python tests/golden/make_golden.py

Each fixture holds float32-representable inputs (cloud, pose, background, d_image) and the
reference outputs: projections, tile lists, pixel state, GradientBuffer, and the parameters after
1 and 10 adam_step calls. They pin the C restatement (tests/test_oracle_pin.py) and the GPU path
(tests/test_gpu_golden.py) on machines without /root/reference.
"""
import os
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle  # noqa: E402
from paper_2404_03202_b200 import scenes  # noqa: E402

FIXTURES = [
    # name, cloud factory, pose, W, H, background
    ("c1_small_uniform", lambda: scenes.synthetic_cloud(1500, seed=21), scenes.identity_pose(), 256, 128,
     (0.0, 0.0, 0.0)),
    ("pole_heavy", lambda: scenes.synthetic_cloud(800, seed=22, variant="pole"), scenes.identity_pose(), 128, 64,
     (0.0, 0.0, 0.0)),
    ("seam_heavy_bg", lambda: scenes.synthetic_cloud(800, seed=23, variant="seam"), scenes.identity_pose(), 128, 64,
     (0.2, 0.3, 0.4)),
    ("random_pose_sh1", lambda: _sh1(), scenes.random_pose(np.random.default_rng(24)), 160, 80, (0.0, 0.0, 0.0)),
]


def _sh1():
    c = scenes.random_cloud(np.random.default_rng(25), count=120, sh_degree=1)
    return c


def main():
    ref = pyoracle.load("reference")
    for name, make, pose, W, H, bg in FIXTURES:
        cloud = make()
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        d_image = rng.uniform(-1.0, 1.0, size=(H, W, 3)).astype(np.float32).astype(np.float64) / (W * H)
        f = ref.render(cloud, pose, W, H, bg, keep_handle=True)
        g = ref.backward(f, d_image, cloud, pose)
        ref.free(f)
        out = dict(positions=cloud.positions, sh=cloud.sh, rotations=cloud.rotations, log_scales=cloud.log_scales,
                   opacity_logits=cloud.opacity_logits, sh_degree=cloud.sh_degree,
                   active_sh_degree=cloud.active_sh_degree, pose=pose, width=W, height=H,
                   background=np.asarray(bg), d_image=d_image, extent=1.25, adam_iterations=30)
        for k, v in dict(gid=f.gaussian_id, p=f.p, conic=f.conic, radius=f.radius, depth=f.depth, color=f.color,
                         offsets=f.offsets, items=f.items, rgb=f.rgb, T=f.T, contributors=f.contributors,
                         last=f.last_contrib).items():
            out["f_" + k] = v
        for k in ("d_position", "d_sh", "d_rotation", "d_log_scale", "d_opacity_logit", "d_screen"):
            out["g_" + k] = getattr(g, k)
        c = cloud.copy()
        st = pyoracle.AdamState.zeros(c.n, c.basis_count)
        cfg = pyoracle.AdamConfig(iterations=30)
        for it in range(1, 11):
            ref.adam_step(c, g, st, cfg, 1.25, it)
            if it in (1, 10):
                for k in ("positions", "sh", "rotations", "log_scales", "opacity_logits"):
                    out[f"adam{it}_{k}"] = getattr(c, k).copy()
        path = os.path.join(HERE, name + ".npz")
        np.savez_compressed(path, **out)
        print(f"{path}: {os.path.getsize(path) / 1e3:.0f} kB, {f.items.size} instances, {f.p.shape[0]} visible")


if __name__ == "__main__":
    main()
