"""C5 check (GPU box): is the Gaussian-count collapse after the first opacity reset the reference's
own behaviour? Trains the roaming scene at reduced size with (a) the reference's own per-step code
(oracle/_ref: render, loss, backward, densify_and_prune, reset_opacity, adam_step, driven by the
Trainer::run restatement in tests/test_gpu_densify.py) on the host cores and (b) osplat_gpu_train on
the GPU, same inputs and config, and prints both Gaussian-count trajectories (one JSON line).

    python scripts/c5_collapse_check.py [--iterations 3400] [--init-points 10000] [--width 380]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import pyoracle  # noqa: E402
from paper_2404_03202_b200 import native, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iterations", type=int, default=3400)
    ap.add_argument("--init-points", type=int, default=10_000)
    ap.add_argument("--gaussians", type=int, default=400_000)
    ap.add_argument("--views", type=int, default=64)
    ap.add_argument("--width", type=int, default=380)
    ap.add_argument("--prune-radius", type=float, default=20.0)
    args = ap.parse_args()
    from test_gpu_densify import oracle_train

    W, H = args.width, args.width // 2
    gt = scenes.roaming_scene(args.gaussians)
    poses = scenes.roaming_poses(args.views)
    gctx = native.Context(gt)
    images = []
    for p in poses:
        fr = gctx.render(p, W, H)
        images.append(fr.image().astype(np.float32).astype(np.float64))
        fr.free()
    gctx.free()
    rng = np.random.default_rng(7)
    pick = rng.choice(gt.n, size=args.init_points, replace=False)
    pts = gt.positions[pick] + rng.normal(0.0, 0.02, (args.init_points, 3))
    rgb = np.clip(gt.sh[pick, 0, :] * 0.28209479177387814 + 0.5, 0.0, 1.0)
    init = scenes.init_from_points(pts, rgb)
    centres = np.array([-(p[:9].reshape(3, 3).T @ p[9:]) for p in poses])
    # scene_extent (trainer.cpp:282-299): 1.1 x the largest camera distance from their mean
    extent = 1.1 * float(np.max(np.linalg.norm(centres - centres.mean(0), axis=1)))
    kw = dict(iterations=args.iterations, log_interval=100, prune_radius_px=args.prune_radius)

    ctx = native.Context(init)
    gpu_log = []
    t0 = time.time()
    ctx.train(native.Config(**kw), poses, images, extent=extent, output_dir="/tmp/c5chk",
              progress=lambda it, loss, n: gpu_log.append((it, loss, n)))
    gpu_s = time.time() - t0

    ref = pyoracle.load("reference")
    ref.set_threads(os.cpu_count() or 1)
    t0 = time.time()
    _, ref_log = oracle_train(ref, init, poses, images, kw, extent)
    ref_s = time.time() - t0
    print(json.dumps({
        "config": f"roaming scene ({gt.n} GT Gaussians), {W}x{H}, {args.views} views, init {init.n} points, "
                  f"reference TrainConfig defaults, prune_radius_px {args.prune_radius}, extent {extent:.3f}",
        "iterations": args.iterations, "gpu_seconds": gpu_s, "reference_seconds": ref_s,
        "reference_threads": ref.threads(),
        "gaussians": [{"iteration": a[0], "gpu": a[2], "reference": b[2], "gpu_loss": a[1], "reference_loss": b[1]}
                      for a, b in zip(gpu_log, ref_log)]}), flush=True)


if __name__ == "__main__":
    main()
