"""Where does the end-to-end train step lose time against the device-timed one? (GPU box)

Times 20 steps of osplat_gpu_train_view + adam_step (wall clock, synchronised) in variants:
host target + loss read-back (the bench's e2e), host target without the read-back, device target
with the read-back, and the device-timed step of bench.py for reference.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2404_03202_b200 import dp, native, scenes  # noqa: E402


def main():
    N, W, H = int(os.environ.get("N", "1000000")), 2048, 1024
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    cloud = scenes.synthetic_cloud(N, seed=1)
    poses = scenes.ring_poses(16, seed=2)
    ctx = native.Context(cloud, stream=stream.cuda_stream)
    fr = ctx.render(poses[0], W, H)
    gt = torch.empty(3 * W * H, dtype=torch.float32, device="cuda")
    gt.copy_(torch.as_tensor(dp._CudaArray(fr.device().rgb, 3 * W * H), device="cuda"))
    fr.free()
    host = torch.empty(3 * W * H, dtype=torch.float32, pin_memory=True)
    host.copy_(gt.cpu())
    cfg = native.Config(iterations=30000)

    def run(label, steps, gt_ptr, on_device, want_loss):
        for it in range(3):
            ctx.train_view(poses[0], W, H, gt_ptr, on_device, 0.2)
            ctx.adam_step(cfg, 1.0, it + 1, zero_grad=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for it in range(steps):
            if want_loss:
                ctx.train_view(poses[0], W, H, gt_ptr, on_device, 0.2)
            else:
                ctx.train_view_noloss(poses[0], W, H, gt_ptr, on_device, 0.2)
            ctx.adam_step(cfg, 1.0, it + 1, zero_grad=True)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / steps * 1e3
        print(f"{label:40s} {ms:7.3f} ms/step", flush=True)

    run("host target + loss read-back", 40, host.data_ptr(), False, True)
    sums = torch.zeros(4, dtype=torch.float64, pin_memory=True)

    def run_async(label, steps, gt_ptr, on_device):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for it in range(steps):
            ctx.train_view_async(poses[0], W, H, gt_ptr, on_device, sums.data_ptr(), 0.2)
            ctx.adam_step(cfg, 1.0, it + 1, zero_grad=True)
        ctx.synchronize()
        ms = (time.perf_counter() - t0) / steps * 1e3
        print(f"{label:40s} {ms:7.3f} ms/step", flush=True)

    run_async("async: host target", 40, host.data_ptr(), False)
    run_async("async: device target", 40, gt.data_ptr(), True)
    # device time of the same step (CUDA events around 40 async steps)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for it in range(40):
        ctx.train_view_async(poses[0], W, H, gt.data_ptr(), True, sums.data_ptr(), 0.2)
        ctx.adam_step(cfg, 1.0, it + 1, zero_grad=True)
    ev1.record(stream)
    ev1.synchronize()
    print(f"{'async device target, CUDA events':40s} {ev0.elapsed_time(ev1) / 40:7.3f} ms/step", flush=True)
    run("host target, no read-back", 20, host.data_ptr(), False, False)
    run("device target + loss read-back", 20, gt.data_ptr(), True, True)
    run("device target, no read-back", 20, gt.data_ptr(), True, False)
    # H2D bandwidth of the pinned target alone
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        gt.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    print(f"{'pinned H2D of the 25 MB target':40s} {(time.perf_counter() - t0) / 20 * 1e3:7.3f} ms")


if __name__ == "__main__":
    main()
