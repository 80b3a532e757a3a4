"""TEST INFRASTRUCTURE: the library's data plane (csrc/comm.cpp) at world 2 on one GPU.

Run with OSPLAT_NCCL_LIB=tests/mock_nccl/libmock_nccl.so (the in-process NCCL stand-in): two
contexts on cuda:0, each driven by its own host thread as rank 0 / rank 1, against one context
that accumulates both ranks' views itself (deterministic backward everywhere). Prints one JSON line.

  1. sharded steps (osplat_gpu_dp_step: reduce-scatter -> Adam on the shard -> all-gather) and a
     densify iteration (screen statistics summed / radii maxed over ranks, moments gathered,
     identical edit on every rank) == the single-process batch computation, bit for bit;
  2. osplat_gpu_train at world 2 (batch of 2 views per iteration, rank 0 writes the files): both
     ranks end with identical parameters.
"""
import json
import os
import sys
import tempfile
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2404_03202_b200 import native, scenes  # noqa: E402

FIELDS = ("positions", "sh", "rotations", "log_scales", "opacity_logits")


def d_images(n, W, H, seed):
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1.0, 1.0, size=(H, W, 3)) / (W * H) for _ in range(n)]


def view_step(ctx, pose, dimg, W, H):
    fr = ctx.render(pose, W, H)
    ctx.backward(fr, dimg, accumulate=True)
    ctx.observe(fr)
    fr.free()


def run_threads(fns):
    errs = []

    def wrap(f):
        try:
            f()
        except BaseException as e:  # surfaced below
            errs.append(repr(e))

    ts = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
    if errs:
        raise RuntimeError("; ".join(errs))


def check_dp_steps():
    W, H = 256, 128
    cloud = scenes.synthetic_cloud(4000, seed=61)
    poses = scenes.ring_poses(4, seed=6)
    dimgs = d_images(4, W, H, 7)
    cfg = native.Config(iterations=100, densify_grad_threshold=1e-7, prune_opacity=0.2)
    world, steps, densify_at = 2, 5, 3

    ref = native.Context(cloud)
    ref.set_deterministic(True)
    ref_summary = None
    for it in range(1, steps + 1):
        for r in range(world):
            v = (world * (it - 1) + r) % 4
            view_step(ref, poses[v], dimgs[v], W, H)
        if it == densify_at:
            ref_summary = ref.densify_and_prune(cfg, 1.0, 77, False)
        else:
            ref.adam_step(cfg, 1.0, it, zero_grad=True)
    want = ref.download()

    uid = native.nccl_unique_id()
    ctxs = [native.Context(cloud) for _ in range(world)]
    summaries = [None] * world

    def rank(r):
        ctx = ctxs[r]
        ctx.set_deterministic(True)
        ctx.dp_init(world, r, uid)
        for it in range(1, steps + 1):
            v = (world * (it - 1) + r) % 4
            view_step(ctx, poses[v], dimgs[v], W, H)
            if it == densify_at:
                summaries[r] = ctx.densify_and_prune(cfg, 1.0, 77, False)
            else:
                ctx.dp_step(cfg, 1.0, it)
        ctx.synchronize()

    run_threads([lambda r=r: rank(r) for r in range(world)])
    got = [c.download() for c in ctxs]
    out = {"ref_summary": ref_summary, "rank_summaries": summaries, "n": [g.n for g in got], "ref_n": want.n}
    out["identical_to_single_process"] = all(
        g.n == want.n and all(np.array_equal(getattr(g, f), getattr(want, f)) for f in FIELDS) for g in got)
    out["max_abs_diff"] = max(float(np.max(np.abs(getattr(g, f) - getattr(want, f)))) if g.n == want.n else -1.0
                              for g in got for f in FIELDS)
    for c in ctxs + [ref]:
        c.free()
    return out


def check_train_world2():
    W, H = 128, 64
    gt = scenes.synthetic_cloud(1500, seed=71)
    cloud = scenes.synthetic_cloud(1200, seed=72)
    rng = np.random.default_rng(8)
    poses = [scenes.random_pose(rng) for _ in range(6)]
    g = native.Context(gt)
    images = []
    for p in poses:
        fr = g.render(p, W, H)
        images.append(fr.image())
        fr.free()
    g.free()
    kw = dict(iterations=24, densify_interval=8, densify_until=20, opacity_reset_interval=12, sh_warmup_interval=6,
              log_interval=6, seed=5, densify_grad_threshold=1e-4)
    world = 2
    uid = native.nccl_unique_id()
    ctxs = [native.Context(cloud) for _ in range(world)]
    tmp = tempfile.mkdtemp()

    def rank(r):
        ctx = ctxs[r]
        ctx.set_deterministic(True)
        ctx.dp_init(world, r, uid)
        ctx.train(native.Config(**kw), poses, images, extent=2.0, output_dir=os.path.join(tmp, f"rank{r}"))
        ctx.synchronize()

    run_threads([lambda r=r: rank(r) for r in range(world)])
    a, b = (c.download() for c in ctxs)
    files = sorted(os.listdir(os.path.join(tmp, "rank0"))) if os.path.isdir(os.path.join(tmp, "rank0")) else []
    out = {"n": [a.n, b.n], "ranks_identical": a.n == b.n and all(np.array_equal(getattr(a, f), getattr(b, f))
                                                                   for f in FIELDS),
           "rank0_files": files,
           "rank1_files": sorted(os.listdir(os.path.join(tmp, "rank1"))) if os.path.isdir(os.path.join(tmp, "rank1"))
           else []}
    for c in ctxs:
        c.free()
    return out


if __name__ == "__main__":
    print(json.dumps({"dp_steps": check_dp_steps(), "train": check_train_world2()}))
