"""GPU probe: element-wise parity of the CUDA path against the reference's own code (oracle/_ref,
all host threads) at the benchmarked sizes. Writes gpurun_out/fullsize_parity.json.

For every case: tile lists, contributors / last_contrib, image, T, then the backward for a
loss-shaped d_image (oracle loss of the oracle render vs a seed-2 target) — per gradient group the
strict-criterion miss count, the max error (relative to the entry and to the group scale) and the
run-to-run spread of the GPU's own gradients (K4a atomics) at the worst entries.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import pyoracle  # noqa: E402
from paper_2404_03202_b200 import native, scenes  # noqa: E402
from parity import compare_tiles  # noqa: E402

GROUPS = ("d_position", "d_sh", "d_rotation", "d_log_scale", "d_opacity_logit")


def grad_report(g, g2, go):
    rep = {}
    for k in GROUPS:
        a = np.asarray(g[k], dtype=np.float64).ravel()
        a2 = np.asarray(g2[k], dtype=np.float64).ravel()
        b = np.asarray(getattr(go, k), dtype=np.float64).ravel()
        scale = max(float(np.max(np.abs(b))), 1e-30)
        err = np.abs(a - b)
        mag = np.maximum(np.abs(a), np.abs(b))
        strict = err > np.maximum(1e-3 * mag, 1e-4 * scale)
        rel = err / np.maximum(mag, 1e-300)
        idx = np.argsort(-(err / np.maximum(1e-3 * mag, 1e-4 * scale)))[:8]
        rep[k] = {"n": int(a.size), "strict_bad": int(strict.sum()), "max_err_over_scale": float(err.max() / scale),
                  "max_rel_above_floor": float(np.max(np.where(mag > 1e-4 * scale, rel, 0.0))),
                  "run_to_run_max_over_scale": float(np.max(np.abs(a - a2)) / scale),
                  "worst": [{"i": int(i), "gpu": float(a[i]), "gpu2": float(a2[i]), "ref": float(b[i]),
                             "err_over_scale": float(err[i] / scale), "rel": float(rel[i])} for i in idx]}
    return rep


def run_case(name, cloud, pose, W, H, oracle, out):
    t0 = time.time()
    ctx = native.Context(cloud)
    fr = ctx.render(pose, W, H)
    t1 = time.time()
    of = oracle.render(cloud, pose, W, H, keep_handle=True)
    t_or = time.time() - t1
    nbad, first = compare_tiles(fr, of)
    rgb, T, con, last = fr.pixels()
    img = fr.image()
    res = {"case": name, "n": cloud.n, "W": W, "H": H, "instances": int(of.items.size),
           "tiles_bad": nbad, "first_bad_tile": first,
           "last_contrib_bad": int(np.sum(last != of.last_contrib)),
           "contributors_bad": int(np.sum(con != of.contributors)),
           "image_max_abs": float(np.max(np.abs(img - of.rgb))),
           "T_max_abs": float(np.max(np.abs(T - of.T))), "oracle_render_s": t_or}
    # loss-shaped d_image: the reference loss gradient of its own render vs a seed-2 target
    tctx = native.Context(scenes.synthetic_cloud(cloud.n, seed=cloud.n % 7 + 2))
    tf = tctx.render(pose, W, H)
    target = tf.image()
    tf.free()
    tctx.free()
    t1 = time.time()
    _, d_image = oracle.loss(of.rgb, target, 0.2, 0.0)
    t2 = time.time()
    go = oracle.backward(of, d_image, cloud, pose)
    res["oracle_loss_s"] = t2 - t1
    res["oracle_backward_s"] = time.time() - t2
    oracle.free(of)
    ctx.backward(fr, d_image)
    g = ctx.gradients()
    ctx.backward(fr, d_image)
    g2 = ctx.gradients()
    res["grads"] = grad_report(g, g2, go)
    res["screen_hits_equal"] = bool(np.array_equal(g["screen_hits"], go.screen_hits))
    ds = np.max(np.abs(go.d_screen))
    res["d_screen_max_over_scale"] = float(np.max(np.abs(g["d_screen"] - go.d_screen)) / max(ds, 1e-30))
    fr.free()
    ctx.free()
    res["wall_s"] = time.time() - t0
    out.append(res)
    print(json.dumps({k: v for k, v in res.items() if k != "grads"}), flush=True)
    for k, v in res["grads"].items():
        print("   ", k, {kk: vv for kk, vv in v.items() if kk != "worst"}, flush=True)


def main():
    which = sys.argv[1:] or ["uniform", "pole", "seam", "opaque", "c4"]
    oracle = pyoracle.load("reference")
    oracle.set_threads(os.cpu_count() or 1)
    out = []
    pose = scenes.ring_poses(16, seed=2)[3]
    for w in which:
        if w == "uniform":
            run_case("1M uniform ring pose 3", scenes.synthetic_cloud(1_000_000, seed=1), pose, 2048, 1024, oracle, out)
        elif w == "pole":
            run_case("1M pole-heavy identity", scenes.synthetic_cloud(1_000_000, seed=1, variant="pole"),
                     scenes.identity_pose(), 2048, 1024, oracle, out)
        elif w == "seam":
            run_case("1M seam-heavy identity", scenes.synthetic_cloud(1_000_000, seed=1, variant="seam"),
                     scenes.identity_pose(), 2048, 1024, oracle, out)
        elif w == "opaque":
            run_case("1M opacity [0.95,0.999] pole-heavy x3 scale",
                     scenes.synthetic_cloud(1_000_000, seed=3, variant="pole", opacity_range=(0.95, 0.999),
                                            scale_mult=3.0), scenes.identity_pose(), 2048, 1024, oracle, out)
            run_case("1M opacity [0.95,0.999] uniform",
                     scenes.synthetic_cloud(1_000_000, seed=4, opacity_range=(0.95, 0.999)), pose, 2048, 1024,
                     oracle, out)
        elif w == "c4":
            run_case("3M uniform 4096x2048 ring pose 3", scenes.synthetic_cloud(3_000_000, seed=1), pose, 4096, 2048,
                     oracle, out)
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", "fullsize_parity.json"), "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
