"""Per-tile load of K3 at 1M / 2048x1024 (uniform and pole-heavy scenes, ring pose 0): list lengths
and visited pairs per tile, per tile row, and a list-scheduling estimate of the K3 tail for the
launch order (blockIdx = row-major tile) vs longest-first. Prints one JSON line per scene."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_03202_b200 import native, scenes  # noqa: E402


def makespan(work, slots, order):
    import heapq
    h = [0.0] * slots
    heapq.heapify(h)
    for t in order:
        s = heapq.heappop(h)
        heapq.heappush(h, s + work[t])
    return max(h)


def main():
    W, H = 2048, 1024
    pose = scenes.ring_poses(16, seed=2)[0]
    for variant in ("uniform", "pole"):
        cloud = scenes.synthetic_cloud(1_000_000, seed=1, variant=variant)
        ctx = native.Context(cloud)
        ctx.profile(timing=False, count_work=True)
        fr = ctx.render(pose, W, H)
        tx, ty, ranges, _ = fr.tiles()
        _, T, con, last = fr.pixels()
        lens = (ranges[:, 1].astype(np.int64) - ranges[:, 0]).reshape(ty, tx)
        # per-tile work proxy: sum over the tile's pixels of the list positions walked
        vis = last.reshape(ty, 16, tx, 16).sum(axis=(1, 3)).astype(np.float64)
        work = lens.astype(np.float64).ravel() * 256.0  # K3 walks the list for every pixel (few stop early)
        slots = 148 * 4
        row_order = np.arange(tx * ty)
        lpt = np.argsort(-work, kind="stable")
        ideal = work.sum() / slots
        out = dict(variant=variant, tiles=int(tx * ty), len_mean=float(lens.mean()), len_max=int(lens.max()),
                   len_row_mean=[round(float(v), 1) for v in lens.mean(axis=1)],
                   last_sum_row=[round(float(v) / 1e6, 3) for v in vis.sum(axis=1)],
                   makespan_rowmajor=makespan(work, slots, row_order) / ideal,
                   makespan_longest_first=makespan(work, slots, lpt) / ideal)
        print(json.dumps(out), flush=True)
        fr.free()


if __name__ == "__main__":
    main()
