"""K4a loop statistics (instrumented build: -DOSB_K4A_STATS, loaded with OSPLAT_LIB=...) for the
1M / 2048x1024 workload of scripts/profile_step.py (ring pose 0). Prints one JSON line."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2404_03202_b200 import dp, native, scenes  # noqa: E402

NAMES = ["sub_visits", "iterations", "iters_with_contrib", "iters_with_tree", "live_halves", "lanes_evaluated",
         "lanes_contributing", "entries_staged"]


def main():
    W, H = 2048, 1024
    cloud = scenes.synthetic_cloud(1_000_000, seed=1)
    poses = scenes.ring_poses(16, seed=2)
    t = native.Context(scenes.synthetic_cloud(1_000_000, seed=2))
    fr = t.render(poses[0], W, H)
    gt = torch.empty(3 * W * H, dtype=torch.float32, device="cuda")
    gt.copy_(torch.as_tensor(dp._CudaArray(fr.device().rgb, 3 * W * H), device="cuda"))
    fr.free()
    ctx = native.Context(cloud)
    lib = native.lib
    lib.osb_k4a_stats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    out = (C.c_ulonglong * 8)()
    lib.osb_k4a_stats(out, 1)
    k3 = (C.c_ulonglong * 5)()
    has_k3 = hasattr(lib, "osb_k3_stats")
    if has_k3:
        lib.osb_k3_stats.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
        lib.osb_k3_stats(k3, 1)
    ctx.profile(timing=False, count_work=True)
    fr = ctx.render(poses[0], W, H)
    ctx.synchronize()
    if has_k3:
        lib.osb_k3_stats(k3, 1)
    _, dimg = ctx.loss(fr, gt.data_ptr(), 0.2, 0.0, want_value=False)
    ctx.backward_device(fr, dimg)
    fwd, bwd, inst = fr.work()
    ctx.synchronize()
    lib.osb_k4a_stats(out, 1)
    st = {n: int(out[i]) for i, n in enumerate(NAMES)}
    st.update(bwd_pairs=bwd, fwd_pairs=fwd, instances=inst)
    if has_k3:
        st.update({f"k3_{n}": int(k3[i]) for i, n in enumerate(
            ["warp_iterations", "lanes_evaluated", "lanes_past_power", "lanes_contributing", "live_halves"])})
    print(json.dumps(st))


if __name__ == "__main__":
    main()
