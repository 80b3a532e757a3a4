"""osplat_render (reference C ABI: host cloud -> host H x W x 3 double image) frames per second at
1M / 2048x1024, wall clock over 40 frames after a warm-up, as bench.py's render e2e (GPU box)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_03202_b200 import native, scenes  # noqa: E402


def main():
    W, H = 2048, 1024
    cloud = scenes.synthetic_cloud(1_000_000, seed=1)
    poses = scenes.ring_poses(16, seed=2)
    hc = native.HostCloud.from_cloud(cloud)
    for k in range(3):
        native.osplat_render(hc, poses[k], W, H)
    nf = 40
    t0 = time.perf_counter()
    for k in range(nf):
        with native.osplat_image(hc, poses[k % 16], W, H) as px:
            float(px[H // 2, ::64].sum())
    print(json.dumps({"osplat_render_fps": nf / (time.perf_counter() - t0)}))


if __name__ == "__main__":
    main()
