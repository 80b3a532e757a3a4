"""GPU: the sharded-optimizer step through real NCCL collectives (world size 1 — the box has one
GPU — with the sharded path forced): in-place reduce_scatter_tensor / all_gather_into_tensor on
views of the flat planes, issued on the context's stream, give the same parameters as the
replicated step."""
import os
import socket

import numpy as np
import pytest

from paper_2404_03202_b200 import dp, native, scenes

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_step_over_nccl_matches_replicated():
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        W, H = 256, 128
        cloud = scenes.synthetic_cloud(5000, seed=21)
        target = scenes.synthetic_cloud(5000, seed=22)
        poses = scenes.ring_poses(4, seed=2)
        tctx = native.Context(target, stream=stream.cuda_stream)
        gts = {}
        for v in range(4):
            fr = tctx.render(poses[v], W, H)
            t = torch.empty(3 * W * H, dtype=torch.float32, device="cuda")
            t.copy_(torch.as_tensor(dp._CudaArray(fr.device().rgb, 3 * W * H), device="cuda"))
            gts[v] = t
            fr.free()
        cfg = native.Config(iterations=100)
        out = []
        for sharded in (False, True):
            ctx = native.Context(cloud, stream=stream.cuda_stream)
            eng = dp.GpuViewEngine(ctx, poses, gts, W, H, cfg)
            if sharded:
                rs, ag = dp.nccl_shard_collectives(dist)
                tr = dp.DataParallelTrainer(eng, 0, 1, reduce_scatter=rs, all_gather=ag, force_shard=True)
                assert tr.sharded
            else:
                tr = dp.DataParallelTrainer(eng, 0, 1)
            for it in range(1, 4):
                tr.step(it, [0, 1, 2, 3])  # 4 views accumulated per step
            torch.cuda.synchronize()
            out.append(ctx.download())
        a, b = out
        for f in ("positions", "sh", "rotations", "log_scales", "opacity_logits"):
            d = np.abs(getattr(a, f) - getattr(b, f))
            # same math; K4a's FP32 atomics reorder sums run to run, which can flip the sign of
            # noise-level gradients (Adam steps them by +-lr)
            assert np.mean(d > 1e-6) < 1e-2, (f, np.mean(d > 1e-6))
            assert np.max(d) <= 3 * 2 * 5e-2, f
    finally:
        dist.destroy_process_group()


def test_densify_exchange_over_nccl_matches_replicated():
    """Training iterations with DensifyStats::observe and a densify iteration (trainer.cpp:364-381)
    through DataParallelTrainer over real NCCL (world 1, sharded path forced: stats allreduce,
    moment all-gather, densify on the replica) == the replicated single-process path, bit for bit
    (deterministic backward on both)."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        W, H = 256, 128
        cloud = scenes.synthetic_cloud(4000, seed=31)
        target = scenes.synthetic_cloud(4000, seed=32)
        poses = scenes.ring_poses(4, seed=3)
        tctx = native.Context(target, stream=stream.cuda_stream)
        gts = {}
        for v in range(4):
            fr = tctx.render(poses[v], W, H)
            t = torch.empty(3 * W * H, dtype=torch.float32, device="cuda")
            t.copy_(torch.as_tensor(dp._CudaArray(fr.device().rgb, 3 * W * H), device="cuda"))
            gts[v] = t
            fr.free()
        cfg = native.Config(iterations=100, densify_grad_threshold=1e-7, prune_opacity=0.2)
        out = []
        for sharded in (False, True):
            ctx = native.Context(cloud, stream=stream.cuda_stream)
            ctx.set_deterministic(True)
            eng = dp.GpuViewEngine(ctx, poses, gts, W, H, cfg, observe=True)
            kw = dict(reduce_stats=dp.nccl_stats_reduce(dist))
            if sharded:
                rs, ag = dp.nccl_shard_collectives(dist)
                tr = dp.DataParallelTrainer(eng, 0, 1, reduce_scatter=rs, all_gather=ag, force_shard=True, **kw)
            else:
                tr = dp.DataParallelTrainer(eng, 0, 1, **kw)
            summary = None
            for it in range(1, 5):
                tr.accumulate([0, 1, 2, 3])
                if it == 2:
                    summary = tr.densify(cfg, 1.0, 77, radius_prune_active=False)
                else:
                    tr.apply(it)
            torch.cuda.synchronize()
            out.append((summary, ctx.download()))
        (s0, a), (s1, b) = out
        assert s0 == s1 and s0["cloned"] + s0["split"] > 0, (s0, s1)
        assert a.n == b.n == s0["final_count"]
        for f in ("positions", "sh", "rotations", "log_scales", "opacity_logits"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
    finally:
        dist.destroy_process_group()


def _gts(stream, W, H, seed, n, poses):
    import torch
    tctx = native.Context(scenes.synthetic_cloud(n, seed=seed), stream=stream.cuda_stream)
    gts = {}
    for v, p in enumerate(poses):
        fr = tctx.render(p, W, H)
        t = torch.empty(3 * W * H, dtype=torch.float32, device="cuda")
        t.copy_(torch.as_tensor(dp._CudaArray(fr.device().rgb, 3 * W * H), device="cuda"))
        gts[v] = t
        fr.free()
    return gts


def test_library_nccl_dp_step_matches_replicated():
    """The library's own data plane (osplat_gpu_dp_init + osplat_gpu_dp_step: ncclReduceScatter ->
    sharded Adam -> ncclAllGather on the context stream, world 1) == the plain Adam step, bit for
    bit, through training steps and a densify iteration (deterministic backward on both)."""
    import torch
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    W, H = 256, 128
    cloud = scenes.synthetic_cloud(4000, seed=41)
    poses = scenes.ring_poses(3, seed=4)
    gts = _gts(stream, W, H, 42, 4000, poses)
    cfg = native.Config(iterations=100, densify_grad_threshold=1e-7, prune_opacity=0.2)
    out = []
    for native_dp in (False, True):
        ctx = native.Context(cloud, stream=stream.cuda_stream)
        ctx.set_deterministic(True)
        if native_dp:
            ctx.dp_init(1, 0, native.nccl_unique_id())
        eng = dp.GpuViewEngine(ctx, poses, gts, W, H, cfg, observe=True)
        tr = dp.DataParallelTrainer(eng, 0, 1, native=native_dp)
        summary = None
        for it in range(1, 5):
            tr.accumulate([0, 1, 2])
            if it == 2:
                summary = tr.densify(cfg, 1.0, 99, radius_prune_active=False)
            else:
                tr.apply(it)
        torch.cuda.synchronize()
        out.append((summary, ctx.download()))
        ctx.free()
    (s0, a), (s1, b) = out
    assert s0 == s1 and s0["cloned"] + s0["split"] > 0
    for f in ("positions", "sh", "rotations", "log_scales", "opacity_logits"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_library_nccl_osplat_gpu_train_world1(tmp_path):
    """osplat_gpu_train on a context with a (world 1) communicator runs the data-parallel loop
    (view stream entry (j-1) world + rank, osplat_gpu_dp_step, collective densify / sidecar) and
    equals the plain Trainer::run bit for bit (deterministic backward)."""
    W, H = 128, 64
    gt = scenes.synthetic_cloud(1500, seed=51)
    cloud = scenes.synthetic_cloud(1200, seed=52)
    rng = np.random.default_rng(6)
    poses = [scenes.random_pose(rng) for _ in range(5)]
    g = native.Context(gt)
    images = []
    for p in poses:
        fr = g.render(p, W, H)
        images.append(fr.image())
        fr.free()
    kw = dict(iterations=30, densify_interval=10, densify_until=25, opacity_reset_interval=15, sh_warmup_interval=8,
              log_interval=5, seed=3, densify_grad_threshold=1e-4)
    res = []
    for k, native_dp in enumerate((False, True)):
        ctx = native.Context(cloud)
        ctx.set_deterministic(True)
        if native_dp:
            ctx.dp_init(1, 0, native.nccl_unique_id())
        log = []
        ctx.train(native.Config(**kw), poses, images, extent=2.0, output_dir=str(tmp_path / f"run{k}"),
                  progress=lambda it, loss, n: log.append((it, loss, n)))
        res.append((log, ctx.download()))
        ctx.free()
    (la, a), (lb, b) = res
    assert la == lb
    for f in ("positions", "sh", "rotations", "log_scales", "opacity_logits"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert open(tmp_path / "run0" / "final.adam", "rb").read() == open(tmp_path / "run1" / "final.adam", "rb").read()
