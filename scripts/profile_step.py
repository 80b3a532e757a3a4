"""Minimal driver for ncu captures: build the 1M / 2048x1024 workload and run a few train steps.

    ncu --set full -k regex:k_blend -s 2 -c 1 -o gpurun_out/blend python scripts/profile_step.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2404_03202_b200 import dp, native, scenes  # noqa: E402


def main():
    n = int(os.environ.get("N", "1000000"))
    W, H = int(os.environ.get("W", "2048")), int(os.environ.get("H", "1024"))
    steps = int(os.environ.get("STEPS", "3"))
    variant = os.environ.get("VARIANT", "uniform")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    cloud = scenes.synthetic_cloud(n, seed=1, variant=variant)
    target = scenes.synthetic_cloud(n, seed=2, variant=variant)
    poses = scenes.ring_poses(16, seed=2)
    tctx = native.Context(target, stream=stream.cuda_stream)
    fr = tctx.render(poses[0], W, H)
    gt = torch.empty(3 * W * H, dtype=torch.float32, device="cuda")
    gt.copy_(torch.as_tensor(dp._CudaArray(fr.device().rgb, 3 * W * H), device="cuda"))
    fr.free()
    del tctx
    ctx = native.Context(cloud, stream=stream.cuda_stream)
    eng = dp.GpuViewEngine(ctx, poses, {0: gt}, W, H, native.Config(iterations=30000))
    tr = dp.DataParallelTrainer(eng, 0, 1)
    for it in range(1, steps + 1):
        tr.step(it, [0])
    torch.cuda.synchronize()
    # the visited pairs of this workload's frame (after the captured launches): the per-pair
    # instruction counts of profiles/ncu_kernels.json divide ncu's totals by these
    ctx.profile(timing=False, count_work=True)
    fr = ctx.render(poses[0], W, H)
    fwd, bwd, inst = fr.work()
    fr.free()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "profile_work.json"), "w") as f:
        json.dump({"gaussians": n, "width": W, "height": H, "variant": variant, "pose": "ring pose 0",
                   "fwd_pairs": fwd, "bwd_pairs": bwd, "instances": inst}, f)
    print("done", native.launch_count(), "launches", fwd, bwd, inst)


if __name__ == "__main__":
    main()
