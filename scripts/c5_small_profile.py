import sys, time, json, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2404_03202_b200 import native, scenes
W, H = 1520, 760
gt = scenes.roaming_scene(300000)
poses = scenes.roaming_poses(40)
g = native.Context(gt)
imgs = []
for p in poses:
    fr = g.render(p, W, H); imgs.append(fr.image()); fr.free()
g.free()
rng = np.random.default_rng(7)
for n in (6000, 30000):
    pick = rng.choice(gt.n, size=n, replace=False)
    init = scenes.init_from_points(gt.positions[pick], np.clip(gt.sh[pick, 0, :] * 0.28209479177387814 + 0.5, 0, 1))
    for prof in (True, False):
        ctx = native.Context(init)
        cfg = native.Config(iterations=2000, mask_bottom_fraction=48/760, log_interval=100000)
        cfg.set("densify_until", 0)
        ctx.profile(timing=prof)
        t = time.time()
        ctx.train(cfg, poses, imgs, is_test=np.zeros(40, np.uint8), extent=0.0, output_dir='/tmp/c5o')
        wall = (time.time() - t) / 2000 * 1e3
        pr = ctx.profile_read()
        print(json.dumps({"n": n, "profiled": prof, "wall_ms": round(wall, 3), "kernel_ms": round(sum(v[0] for v in pr.values()) / 2000, 3)}))
        ctx.free()
