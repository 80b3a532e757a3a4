"""Per-kernel render time of the pole-heavy and uniform C3 scenes (GPU box)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_03202_b200 import native, scenes  # noqa: E402

for variant in ("uniform", "pole"):
    ctx = native.Context(scenes.synthetic_cloud(1_000_000, seed=1, variant=variant))
    pose = scenes.identity_pose()
    for _ in range(3):
        ctx.render(pose, 2048, 1024).free()
    ctx.profile(timing=True)
    for _ in range(10):
        ctx.render(pose, 2048, 1024).free()
    pr = ctx.profile_read()
    print(json.dumps({"variant": variant, "ms_per_frame": {k: round(v[0] / 10, 4) for k, v in pr.items() if v[1]}}))
    ctx.free()
