#!/usr/bin/env python
"""bench.py — "ERP render FPS + fwd/bwd train iters/s, 1M Gaussians at 2048x1024" (BASELINE.json).

One step = one training iteration of the hot path on every GPU: per view, render (K1 preprocess ->
K2 depth/tile sort -> K3 blend) -> loss (L1 + SSIM, lambda 0.2) -> backward (K4a pixels -> K4b
Gaussians, accumulate), then (N > 1) the NCCL reduce-scatter of the flat gradient planes, the fused
Adam step (K5) on this rank's shard and the all-gather of the parameters.
Weak scaling by default: every GPU trains `--views-per-gpu` views per iteration on the replicated
1M-Gaussian scene; `--global-views B` instead fixes the batch at B views split over the GPUs
(strong scaling). Views cycle over 16 ring poses; `value` = views trained per
second over the whole job (= train iterations/s at N = 1). `render_fps` = K1 -> K3 frames/s.

    python bench.py [--gpus N --steps K --warmup W]    # our arm; N > 1 spawns N ranks itself when
                                                       # not launched by torchrun
    python bench.py --impl reference [...]             # the reference CPU code on the host cores

Prints ONE JSON line on rank 0. Inputs are synthetic (scenes.synthetic_cloud, seed 1; the loss
target of each view is a render of the seed-2 scene from that view).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ERP render FPS + fwd/bwd train iters/s, 1M Gaussians at 2048x1024"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}
N_POSES = 16
LAMBDA_SSIM = 0.2  # TrainConfig default (trainer.hpp:20), both arms
SMS, SMSP_PER_SM = 148, 4  # B200: 148 SMs x 4 sub-partitions, one warp instruction issued per cycle each


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--gaussians", type=int, default=1_000_000)
    p.add_argument("--width", type=int, default=2048)
    p.add_argument("--height", type=int, default=1024)
    p.add_argument("--views-per-gpu", type=int, default=1)
    p.add_argument("--global-views", type=int, default=0,
                   help="fixed batch of B views per step split over the GPUs (strong scaling); 0 = weak")
    p.add_argument("--torch-collectives", action="store_true",
                   help="N > 1: exchange through torch.distributed (NCCL) instead of the library's own NCCL calls")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-sweep", action="store_true", help="skip the render FPS sweep (pole/seam scenes)")
    return p.parse_args()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                "source": "measured (MEASURED_PEAKS.json)"}
    return dict(PEAKS_FALLBACK)


def load_ncu_kernels():
    """Per kernel family, from one ncu --set full capture of the same workload (profiles/): warp
    instructions and DRAM bytes per launch, issue-active / FMA-pipe %, and the visited pairs of that
    launch's frame (scripts/ncu_kernels.py)."""
    path = os.path.join(ROOT, "profiles", "ncu_kernels.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


# ------------------------------------------------------------------------------------------------

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def views_per_rank(args, world):
    if args.global_views:
        if args.global_views % world:
            raise SystemExit(f"bench.py: --global-views {args.global_views} is not a multiple of {world} GPUs")
        return args.global_views // world
    return args.views_per_gpu


def step_views(step: int, rank: int, world: int, V: int) -> list:
    """The views rank `rank` trains in step `step`: the global batch of world * V consecutive ring
    poses (cycling over the 16), view j of the batch on rank j % world (dp.views_for_rank)."""
    from paper_2404_03202_b200 import dp
    return dp.views_for_rank(step, world * V, N_POSES, rank, world)


def workload_config(args, world, V):
    scaling = (f"strong: {args.global_views} views per step split over the GPUs" if args.global_views else
               f"weak: {V} view(s) per GPU per step")
    return {"workload": f"{args.gaussians // 1000}k Gaussians, {args.width}x{args.height} ERP, train step "
                        f"(render + L1+SSIM loss + backward + Adam), {scaling}",
            "gaussians": args.gaussians, "width": args.width, "height": args.height,
            "views_per_gpu_per_step": V, "global_batch_views": world * V, "poses": f"{N_POSES} ring poses, cycled",
            "sh_degree": 3, "scene": "synthetic uniform shell, seed 1; targets: seed-2 scene rendered per view",
            "lambda_ssim": LAMBDA_SSIM,
            "parallelism": f"dp{world} (views split, Gaussians replicated; N > 1: NCCL reduce-scatter of the "
                           f"gradients, sharded Adam, all-gather of the parameters)",
            "l2": f"inputs larger than L2: params + grads + Adam moments = 4 x "
                  f"{args.gaussians * 59 * 4 / 1e6:.0f} MB resident"}


# ------------------------------------------------------------------------------------------------ reference arm

def reference_oracle(threads=None):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    kind = "reference" if pyoracle.available("reference") else "port"
    o = pyoracle.load(kind)
    o.set_threads(threads or os.cpu_count() or 1)
    return o, kind, o.threads()


def cpu_reference_step(oracle, cloud, pose, gt, W, H, cfg, it):
    """One reference train step (render + loss + backward + adam_step), the reference's own
    steady-clock time of each call summed (eval.cpp:84-87 convention; marshalling excluded).
    Returns (seconds, render seconds)."""
    import pyoracle
    f = oracle.render(cloud, pose, W, H, keep_handle=True)
    t_render = oracle.last_seconds()
    t = t_render
    _, d = oracle.loss(f.rgb, gt, LAMBDA_SSIM, 0.0)
    t += oracle.last_seconds()
    g = oracle.backward(f, d, cloud, pose)
    t += oracle.last_seconds()
    oracle.free(f)
    st = pyoracle.AdamState.zeros(cloud.n, cloud.basis_count)
    oracle.adam_step(cloud, g, st, cfg, 1.0, it)
    t += oracle.last_seconds()
    return t, t_render


def run_reference_arm(args):
    """The reference's own CPU implementation (oracle/_ref: the reference sources compiled by
    oracle/Makefile) on all host threads; rank 0 alone under torchrun. Same config, views, targets
    (the seed-2 scene rendered by the reference itself), warm-up and step count as our arm."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2404_03202_b200 import scenes  # numpy only: this process never maps the product library
    oracle, kind, cores = reference_oracle()
    import pyoracle
    N, W, H = args.gaussians, args.width, args.height
    G = max(args.gpus, world)
    V = views_per_rank(args, G)
    cloud = scenes.synthetic_cloud(N, seed=1)
    target_cloud = scenes.synthetic_cloud(N, seed=2)
    poses = scenes.ring_poses(N_POSES, seed=2)
    targets = {}
    cfg = pyoracle.AdamConfig(iterations=30000)
    warm = max(args.warmup, 3)
    times, rtimes = [], []
    budget, t_start = 300.0, time.time()
    # one reference iteration = one view (trainer.cpp:353-381); its per-view cost does not depend on
    # how many GPUs our arm splits the batch over, so the host runs the batch's views one after the
    # other and views/s is the comparable rate
    for i in range(warm + args.steps):
        vi = i % N_POSES
        if vi not in targets:
            targets[vi] = oracle.render(target_cloud, poses[vi], W, H).rgb
        t, tr = cpu_reference_step(oracle, cloud, poses[vi], targets[vi], W, H, cfg, i + 1)
        if i >= warm:
            times.append(t)
            rtimes.append(tr)
        if time.time() - t_start > budget and len(times) >= 1:
            break
    sec = float(np.mean(times))
    value = 1.0 / sec
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "views/s", "n_gpus": G,
            "steps": args.steps, "steps_run": len(times), "warmup": warm, "ms_per_step": sec * 1e3,
            "train_iters_per_s": value,
            "higher_is_better": True, "scaling": "strong" if args.global_views else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": workload_config(args, G, V),
            "render_fps": 1.0 / float(np.mean(rtimes)),
            "cpu_baseline": {"value": value, "unit": "views/s", "cores": cores, "kind": kind, "cpu": cpu_model(),
                             "sample": f"{len(times)} full train step(s) of one view of the workload on the host "
                                       f"(reference render + loss + backward + adam_step, steady clock, cycling "
                                       f"the {N_POSES} ring poses; targets = the seed-2 scene rendered by the "
                                       f"reference)"},
            "e2e": {"value": value, "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baselines(gpu_target_img, W, H, N, pose):
    """The reference on this host (rank 0, N = 1), bounded: the workload's train step on all
    threads, and SURVEY §8(d)'s C1 (10k, 512x256) / C2 (100k, 1024x512) steps on 1 thread and on all
    threads. Returns the cpu_baseline object."""
    from paper_2404_03202_b200 import scenes
    oracle, kind, cores = reference_oracle()
    import pyoracle
    cfg = pyoracle.AdamConfig(iterations=30000)
    cloud = scenes.synthetic_cloud(N, seed=1)
    secs, rsecs = cpu_reference_step(oracle, cloud, pose, gpu_target_img, W, H, cfg, 1)
    out = {"value": 1.0 / secs, "unit": "views/s", "cores": cores, "kind": kind, "cpu": cpu_model(),
           "sample": f"1 full train step of the workload ({N // 1000}k, {W}x{H}: reference render + loss + "
                     f"backward + adam_step, steady clock, marshalling excluded) on {cores} threads",
           "seconds": secs, "render_fps": 1.0 / rsecs, "configs": {}}
    for name, n, w, h, threads in (("C1_10k_512x256", 10_000, 512, 256, 1), ("C1_10k_512x256", 10_000, 512, 256, cores),
                                   ("C2_100k_1024x512", 100_000, 1024, 512, 1),
                                   ("C2_100k_1024x512", 100_000, 1024, 512, cores)):
        oracle.set_threads(threads)
        c = scenes.synthetic_cloud(n, seed=1)
        gt = oracle.render(scenes.synthetic_cloud(n, seed=2), pose, w, h).rgb
        s, r = cpu_reference_step(oracle, c, pose, gt, w, h, cfg, 1)
        out["configs"][f"{name}_{threads}t"] = {"train_step_s": s, "render_s": r, "threads": threads}
    oracle.set_threads(cores)
    return out


# ------------------------------------------------------------------------------------------------ our arm

class CudaArray:
    """Minimal __cuda_array_interface__ wrapper so torch can view our device buffers zero-copy."""

    def __init__(self, ptr, n, typestr="<f4"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def run_ours(args):
    rank, world, local = dist_env()
    if os.environ.get("OSPLAT_BENCH_DRYRUN"):  # launcher test (tests/test_bench_cpu.py): report and exit
        print(json.dumps({"rank": rank, "world": world, "local_rank": local, "gpus": args.gpus,
                          "master": f"{os.environ.get('MASTER_ADDR')}:{os.environ.get('MASTER_PORT')}"}), flush=True)
        return
    import torch
    import torch.distributed as dist
    from paper_2404_03202_b200 import dp, native, scenes

    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product has no CPU path)")
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local}, {torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    nccl = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        nccl = {"backend": dist.get_backend(), "comm_nranks": dist.get_world_size(),
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
    # one dedicated stream for everything: our kernels (the context adopts it), NCCL (torch waits on
    # the current stream) and the timing events
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    N, W, H = args.gaussians, args.width, args.height
    V = views_per_rank(args, world)
    peaks = load_peaks()
    plane = W * H

    cloud = scenes.synthetic_cloud(N, seed=1)
    poses = scenes.ring_poses(N_POSES, seed=2)
    my_views = sorted({v for s in range(N_POSES) for v in step_views(s, rank, world, V)})

    # loss targets: renders of the seed-2 scene from each of this rank's views, device resident
    gts = {}
    tctx = native.Context(scenes.synthetic_cloud(N, seed=2), device=local, stream=stream.cuda_stream)
    for vi in my_views:
        fr = tctx.render(poses[vi], W, H)
        t = torch.empty(3 * plane, dtype=torch.float32, device="cuda")
        t.copy_(torch.as_tensor(CudaArray(fr.device().rgb, 3 * plane), device="cuda"))
        gts[vi] = t
        fr.free()
    tctx.synchronize()
    tctx.free()

    ctx = native.Context(cloud, device=local, stream=stream.cuda_stream)
    cfg = native.Config(iterations=30000)
    extent = 1.0
    engine = dp.GpuViewEngine(ctx, poses, gts, W, H, cfg, extent, lambda_ssim=LAMBDA_SSIM)
    # N > 1: sharded optimizer — reduce-scatter of the gradient planes, fused Adam on this rank's
    # 1/N shard, all-gather of the parameters, in place on the flat buffers on `stream`. Default: the
    # library's own NCCL communicator (osplat_gpu_dp_init / osplat_gpu_dp_step; torch.distributed
    # only hands out the unique id); --torch-collectives: the same exchange through torch.distributed.
    coll_ms = []
    timing_coll = [False]
    native_dp = world > 1 and not args.torch_collectives
    rs = ag = None
    if native_dp:
        uid = [native.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.dp_init(world, rank, uid[0])
        nccl["data_plane"] = "libosplat_b200 (ncclCommInitRank + ncclReduceScatter / ncclAllGather on the context stream)"
    elif world > 1:
        rs, ag = dp.nccl_shard_collectives(dist)
        nccl["data_plane"] = "torch.distributed (reduce_scatter_tensor / all_gather_into_tensor)"

    class TimedEngine:
        """Times each exchange (reduce-scatter + sharded Adam + all-gather) with events on `stream`."""

        def __getattr__(self, name):
            return getattr(engine, name)

        def _timed(self, fn, *a):
            if not timing_coll[0]:
                return fn(*a)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(*a)
            e1.record(stream)
            coll_ms.append((e0, e1))

        def dp_step(self, iteration):
            self._timed(engine.dp_step, iteration)

    if world > 1 and not native_dp:
        rs0, ag0 = rs, ag

        def rs(t, b, c):
            if timing_coll[0]:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                coll_ms.append([e0, None])
            rs0(t, b, c)

        def ag(t, b, c):
            ag0(t, b, c)
            if timing_coll[0]:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                coll_ms[-1][1] = e1
    trainer = dp.DataParallelTrainer(TimedEngine(), rank, world, reduce_scatter=rs, all_gather=ag, native=native_dp)
    step_idx = [0]

    def train_step():
        trainer.step(step_idx[0] + 1, step_views(step_idx[0], rank, world, V))
        step_idx[0] += 1

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    warm = max(args.warmup, 3)
    for _ in range(warm):
        train_step()
    barrier()
    # clocks are sampled from here to the end of the profiled pass; keep the GPU busy for ~0.6 s
    # first so the sampler sees the steady state of this load
    clocks = ClockSampler(local)
    clocks.start()
    t_warm = time.perf_counter()
    while time.perf_counter() - t_warm < 0.6:
        train_step()
        torch.cuda.synchronize()
    barrier()

    # ---- timed train steps (device time, CUDA events on the launching stream, no profiler)
    first_step = step_idx[0]
    launches0 = native.launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev[0].record(stream)
    for k in range(args.steps):
        train_step()
        ev[k + 1].record(stream)
    barrier()
    ms_total = max_over_ranks(ev[0].elapsed_time(ev[-1]))
    step_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    print(f"[bench] step ms: {['%.2f' % x for x in step_ms]}", file=sys.stderr, flush=True)
    launches = native.launch_count() - launches0
    ms_per_step = ms_total / args.steps
    value = world * V * args.steps / (ms_total / 1e3)

    # ---- the same view sequence again with per-kernel CUDA events (roofline evidence)
    step_idx[0] = first_step
    ctx.profile(timing=True, count_work=False)
    ctx.profile_read(reset=True)
    timing_coll[0] = True
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        train_step()
    p1.record(stream)
    barrier()
    timing_coll[0] = False
    ms_profiled = p0.elapsed_time(p1)
    prof = ctx.profile_read(reset=True)
    ctx.profile(timing=False)
    clk = clocks.stop()
    collectives = None
    if world > 1:
        flat_bytes = engine.grad_tensor().numel() * 4
        ms = float(np.mean([a.elapsed_time(b) for a, b in coll_ms])) if coll_ms else None
        collectives = dict(nccl)
        # reduce-scatter + all-gather move the bytes of one ring allreduce: 2 (N - 1) / N x buffer
        collectives["exchange"] = {"ms_per_step": ms, "buffer_bytes": flat_bytes,
                                   "what": "reduce-scatter of the gradient planes + fused Adam on the 1/N shard + "
                                           "all-gather of the parameters",
                                   "bus_gbs": 2 * (world - 1) / world * flat_bytes / (ms / 1e3) / 1e9 if ms else None}

    # work counts of the profiled views (untimed renders with the device counters on)
    fwd_pairs = bwd_pairs = instances = 0
    ctx.profile(timing=False, count_work=True)
    for s in range(first_step, first_step + args.steps):
        for vi in step_views(s, rank, world, V):
            fr = ctx.render(poses[vi], W, H)
            fp, bp, inst = fr.work()
            fr.free()
            fwd_pairs, bwd_pairs, instances = fwd_pairs + fp, bwd_pairs + bp, instances + inst
    ctx.profile(timing=False, count_work=False)
    nviews = args.steps * V
    fwd_pairs, bwd_pairs, instances = fwd_pairs / nviews, bwd_pairs / nviews, instances / nviews
    ctx.zero_grad()

    # ---- render-only FPS (K1 -> K3), device time: the synthetic scene as generated (a fresh context
    # holding the seed-1 cloud the training started from), so the number does not depend on how
    # many train steps ran before it
    barrier()
    rctx = native.Context(cloud, device=local, stream=stream.cuda_stream)
    for k in range(3):
        rctx.render(poses[k % N_POSES], W, H).free()
    nframes = max(args.steps, 4 * N_POSES)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    for k in range(nframes):
        rctx.render(poses[k % N_POSES], W, H).free()
    r1.record(stream)
    barrier()
    render_ms = max_over_ranks(r0.elapsed_time(r1)) / nframes
    # the same frames again with per-kernel CUDA events (the split; its total includes the events)
    rctx.profile(timing=True)
    rctx.profile_read(reset=True)
    for k in range(nframes):
        rctx.render(poses[k % N_POSES], W, H).free()
    barrier()
    rprof = rctx.profile_read(reset=True)
    rctx.profile(timing=False)

    # ---- render FPS sweep (BASELINE configs[2]): the uniform scene over 36 yaws x pitch {0, +-60 deg},
    # and the pole-heavy (|lat| > 70 deg) and seam-heavy (|lon| > 160 deg) scenes over 12 yaws;
    # per-frame device time (CUDA events), median and 5th-percentile FPS per variant
    sweep = None
    if rank == 0 and not args.no_sweep:
        def frame_ms(c, poses_list):
            out = []
            for p in poses_list:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                c.render(p, W, H).free()
                b.record(stream)
                b.synchronize()
                out.append(a.elapsed_time(b))
            return out

        def summary(ms):
            fps = sorted(1e3 / np.asarray(ms))
            return {"frames": len(ms), "fps_median": float(np.median(fps)), "fps_p5": float(np.percentile(fps, 5)),
                    "ms_median": float(np.median(ms))}

        yaw_pitch = [scenes.pose12(scenes.rot_x(np.radians(pt)) @ scenes.rot_y(np.radians(yw)))
                     for pt in (0.0, 60.0, -60.0) for yw in range(0, 360, 10)]
        frame_ms(rctx, yaw_pitch[:3])
        sweep = {"uniform_36yaw_x3pitch": summary(frame_ms(rctx, yaw_pitch))}
        for variant in ("pole", "seam"):
            vc = native.Context(scenes.synthetic_cloud(N, seed=1, variant=variant), device=local,
                                stream=stream.cuda_stream)
            vc.profile(timing=False, count_work=True)
            fr = vc.render(scenes.identity_pose(), W, H)
            fp, bp, inst = fr.work()
            fr.free()
            vc.profile(timing=False, count_work=False)
            views = [scenes.pose12(scenes.rot_y(np.radians(yw))) for yw in range(0, 360, 30)]
            frame_ms(vc, views[:2])
            sweep[f"{variant}_heavy_12yaw"] = dict(summary(frame_ms(vc, views)), instances=inst, fwd_pairs=fp)
            vc.free()
    rctx.free()

    # ---- end to end through the public C ABI with host buffers
    e2e = None
    render_e2e = None
    if not args.no_e2e:
        host_gt = {vi: torch.empty(3 * plane, dtype=torch.float32, pin_memory=True) for vi in my_views}
        for vi in my_views:
            host_gt[vi].copy_(gts[vi].cpu())
        e2e_steps = max(3 * args.steps, 30)  # wall clock: enough steps to average out host jitter
        # pinned slots for every step's loss sums: each step's D2H read is enqueued (async), the
        # host waits once at the end of the timed region and turns every step's sums into its loss
        sums_host = torch.zeros((e2e_steps + warm + 8, V, 4), dtype=torch.float64, pin_memory=True)
        losses = []
        grads = engine.grad_tensor()

        def e2e_step():
            s = step_idx[0]
            slot = sums_host[len(losses) % sums_host.shape[0]]
            views = step_views(s, rank, world, V)
            losses.append(slot)
            for k, vi in enumerate(views):
                ctx.train_view_async(poses[vi], W, H, host_gt[vi].data_ptr(), gt_on_device=False,
                                     sums_ptr=slot[k].data_ptr(), lambda_ssim=LAMBDA_SSIM)
            if native_dp:
                ctx.dp_step(cfg, extent, s + 1)
            elif world > 1:
                b0, cnt = dp.shard_range(grads.numel(), rank, world)
                rs(grads, b0, cnt)
                ctx.adam_step(cfg, extent, s + 1, zero_grad=True, begin=b0, count=cnt)
                ag(engine.param_tensor(), b0, cnt)
            else:
                ctx.adam_step(cfg, extent, s + 1, zero_grad=True)
            step_idx[0] += 1

        for _ in range(warm):  # first use creates the copy stream and the target buffer
            e2e_step()
        barrier()
        ctx.synchronize()
        losses.clear()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        ctx.synchronize()  # every step's loss sums are on the host now
        step_losses = [sum(native.loss_value(slot[k].numpy(), LAMBDA_SSIM, W, H) for k in range(V))
                       for slot in losses]
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        assert all(np.isfinite(step_losses)), "non-finite loss in the e2e run"
        e2e = {"value": world * V * e2e_steps / e2e_s, "unit": "views/s", "steps": e2e_steps,
               "h2d_bytes_per_step": V * 3 * plane * 4, "d2h_bytes_per_step": V * 32,
               "loss_first_last": [step_losses[0], step_losses[-1]],
               "api": "osplat_gpu_train_view_async per view (pinned host target in, loss sums out to pinned host "
                      "every step, one wait at the end) + osplat_gpu_adam_step (N > 1: osplat_gpu_dp_step = NCCL "
                      "reduce-scatter + sharded Adam + all-gather inside the library)"}
        if rank == 0:
            hc = native.HostCloud.from_cloud(cloud)
            native.osplat_render(hc, poses[0], W, H)  # upload + warm
            t0 = time.perf_counter()
            nf = max(3, min(args.steps, 10))
            checks = []
            for k in range(nf):
                with native.osplat_image(hc, poses[k % N_POSES], W, H) as px:  # osplat_render .. _free
                    checks.append(float(px[H // 2, ::64].sum()))  # read the host image
            render_e2e = {"value": nf / (time.perf_counter() - t0), "unit": "FPS",
                          "api": "osplat_render + osplat_image_pixels + osplat_image_free (reference C ABI: host "
                                 "cloud -> host H x W x 3 double image)",
                          "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 3 * plane * 8}
            assert all(np.isfinite(checks))

    # ---- rooflines of the kernel families in the profiled train steps
    clk_mhz = peaks["sm_max_mhz"]
    issue_peak = SMS * SMSP_PER_SM * clk_mhz * 1e6 / 1e12  # T warp-instructions / s
    ncu = load_ncu_kernels()
    per_launch_ms = {k: v[0] / max(v[1], 1) for k, v in prof.items() if v[1]}
    launches_per_view = {k: v[1] / nviews for k, v in prof.items() if v[1]}
    planes = engine.grad_tensor().numel()
    # algorithmic bytes per launch; K3/K4a: pairs x the kernel's measured warp
    # instructions per pair (ncu, profiles/ncu_kernels.json) -> issue-slot utilisation
    hbm = {
        # K1: the 59 parameter planes (236 B) in, the frame's per-Gaussian records out — depth keys 12,
        # touched 4, rectangle 16, FP64 centre 16 + conic/opacity 32, FP32 blend record 48, radius 4 =
        # 132 B per visible Gaussian (upper bound: every Gaussian counted as visible)
        "preprocess": N * (236 + 132),
        "depth_sort": N * 12 * 2 * 8,
        # two 8-byte (tile, id) passes in and out; the last pass stores ids only (its keys become the
        # tile ranges): 8 + 8 + 8 + 4 = 28 B per instance
        "tile_sort": instances * 28,
        "loss": plane * 36,
        # K4b per visible Gaussian: parameters 236 + K4a accumulators 48 + K1 records (conic 32, blend
        # record 48, depth key 8) in; gradient planes 236 + screen statistics 20 out (upper bound)
        "bwd_gauss": N * (236 + 48 + 88 + 236 + 20),
        "adam": 28 * planes / world,  # p, g, m, v in, p, m, v out (N > 1: this rank's 1/N shard)
    }
    pairs = {"blend": fwd_pairs, "bwd_pixels": bwd_pairs}
    rooflines = {}
    for name, ms in per_launch_ms.items():
        k = ncu.get(name, {})
        ent = {"ms_per_launch": ms, "share_of_step": prof[name][0] / max(ms_profiled, 1e-9),
               "traffic": k.get("dram_bytes"), "ncu_issue_active": k.get("issue_active_pct"),
               "ncu_fma_pipe": k.get("fma_pipe_pct")}
        if name in pairs and k.get("warp_instructions") and k.get("pairs"):
            ipp = k["warp_instructions"] / k["pairs"]  # warp instructions per visited pair (ncu)
            units = pairs[name] / launches_per_view[name]
            achieved = units * ipp / (ms / 1e3) / 1e12
            ent.update(bound="issue", achieved=achieved, peak=issue_peak, unit="T warp-instr/s",
                       frac=achieved / issue_peak, pairs_per_launch=units, warp_instr_per_pair=ipp)
        elif name in hbm:
            achieved = hbm[name] / launches_per_view[name] / (ms / 1e3) / 1e9
            ent.update(bound="hbm", achieved=achieved, peak=peaks["hbm_gbs"], unit="GB/s",
                       frac=achieved / peaks["hbm_gbs"], algorithmic_bytes=hbm[name] / launches_per_view[name])
        rooflines[name] = ent
    dominant = max(per_launch_ms, key=lambda k: prof[k][0])
    roof = dict(rooflines.get(dominant, {}))
    roof["kernel"] = dominant
    if roof.get("bound") == "issue":
        roof["peak_source"] = (f"instruction issue: {SMS} SMs x {SMSP_PER_SM} sub-partitions x 1 warp-instr/clk x "
                               f"{clk_mhz:.0f} MHz (derived)")
        roof["note"] = ("K3/K4a are neither HBM- nor tensor-bound (no dense contraction; SURVEY 8(d)); the bound is "
                        "instruction issue. achieved = visited (pixel, splat) pairs per launch (counted on the "
                        "device, this run) x warp instructions per pair (ncu --set full of the same workload, "
                        "profiles/ncu_kernels.json) / live CUDA-event launch time")
    else:
        roof["peak_source"] = peaks["source"]

    # ---- CPU baseline (rank 0, N == 1): the reference code on this host's cores
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v0 = step_views(first_step, 0, 1, V)[0]
            gt_host = gts[v0].cpu().numpy().reshape(3, H, W).transpose(1, 2, 0).astype(np.float64)
            cpu = cpu_baselines(gt_host, W, H, N, poses[v0])
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "views/s", "cores": os.cpu_count(), "kind": "unavailable",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "views/s", "n_gpus": world, "steps": args.steps,
                "warmup": warm, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if args.global_views else "weak", "vs_baseline": None,
                "dtype": "f32 (f64 geometry + guard)", "data": "synthetic", "config": workload_config(args, world, V),
                "train_iters_per_s": value / (world * V),
                "render_fps": 1e3 / render_ms,
                "render": {"ms_per_frame": render_ms, "frames": nframes,
                           "kernels_ms_per_frame": {k: v[0] / nframes for k, v in rprof.items() if v[1]},
                           "e2e": render_e2e, "sweep": sweep},
                "work_per_view": {"fwd_pairs": fwd_pairs, "bwd_pairs": bwd_pairs, "instances": instances},
                "kernels_ms_per_step": {k: v[0] / args.steps for k, v in prof.items() if v[1]},
                "ms_per_step_profiled": ms_profiled / args.steps,
                "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
                "collectives": collectives,
                "roofline": roof, "rooflines": rooflines, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk}
        print(json.dumps(line), flush=True)
    ctx.free()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: one process per GPU, launched here with the torchrun
    environment (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR=127.0.0.1 / MASTER_PORT)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus), LOCAL_WORLD_SIZE=str(args.gpus),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
