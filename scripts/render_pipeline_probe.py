"""Render throughput with two frames in flight (GPU box): two contexts holding the same cloud on two
streams render alternate poses, so one frame's K1 / K2 (latency-bound, low issue utilisation) can
overlap the other's K3. Compared with one context rendering the same poses back to back. Device
time with CUDA events. Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2404_03202_b200 import native, scenes  # noqa: E402


def main():
    W, H = 2048, 1024
    n = int(os.environ.get("N", "1000000"))
    variant = os.environ.get("VARIANT", "uniform")
    cloud = scenes.synthetic_cloud(n, seed=1, variant=variant)
    poses = scenes.ring_poses(16, seed=2)
    frames = 64
    out = {"variant": variant}
    for prio in (0, -1):
        s0 = torch.cuda.Stream(priority=0)
        s1 = torch.cuda.Stream(priority=prio)
        ctx = [native.Context(cloud, stream=s0.cuda_stream), native.Context(cloud, stream=s1.cuda_stream)]
        for c in ctx:
            for p in poses[:3]:
                c.render(p, W, H).free()
        torch.cuda.synchronize()
        # one context, back to back
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s0)
        for i in range(frames):
            ctx[0].render(poses[i % 16], W, H).free()
        e1.record(s0)
        torch.cuda.synchronize()
        serial = e0.elapsed_time(e1) / frames
        # two contexts, alternating, two frames in flight
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s0)
        s1.wait_event(a)
        live = []
        for i in range(frames):
            live.append(ctx[i % 2].render(poses[i % 16], W, H))
            if len(live) > 2:
                live.pop(0).free()
        for f in live:
            f.free()
        done1 = torch.cuda.Event()
        done1.record(s1)
        s0.wait_event(done1)
        b.record(s0)
        torch.cuda.synchronize()
        piped = a.elapsed_time(b) / frames
        out[f"prio{prio}"] = {"serial_ms": serial, "serial_fps": 1e3 / serial, "pipelined_ms": piped,
                              "pipelined_fps": 1e3 / piped}
        for c in ctx:
            c.free()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
