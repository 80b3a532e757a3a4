"""Build profiles/ncu_kernels.json — what bench.py's roofline reads — from an ncu summary
(scripts/ncu_summary.py --json) and the workload's work counts (gpurun_out/profile_work.json,
written by scripts/profile_step.py for the same frame).

    python scripts/ncu_kernels.py profiles/ncu_summary_r02.json gpurun_out/profile_work.json

Per kernel family (bench.py's names): warp instructions, DRAM bytes read + written, duration,
issue-active %, FMA-pipe %, and for K3 / K4a the visited pairs of the captured launch.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAMILY = {"k_backward_pixels": "bwd_pixels", "k_blend": "blend", "k_preprocess": "preprocess", "k_adam": "adam",
          "k_backward_gaussians": "bwd_gauss", "k_ssim_fwd": "loss", "k_ssim_bwd": "loss_bwd"}


def main():
    summary = json.load(open(sys.argv[1]))
    work = json.load(open(sys.argv[2]))
    out = {"_source": f"{os.path.basename(sys.argv[1])} (ncu --set full --clock-control none, one launch per kernel "
                      f"inside scripts/profile_step.py) + work counts of the same frame {work}"}
    for name, d in summary.items():
        short = name.replace("void ", "").replace("unnamed>::", "").split("<")[0].strip()
        fam = FAMILY.get(short)
        if not fam:
            continue
        ent = {"kernel": short, "warp_instructions": d.get("warp_instructions"),
               "dram_bytes": (d.get("dram_read", 0) + d.get("dram_write", 0)) * (1e6 if d.get("dram_read_unit") == "Mbyte" else
                                                                                   1e9 if d.get("dram_read_unit") == "Gbyte" else
                                                                                   1e3 if d.get("dram_read_unit") == "Kbyte" else 1),
               "duration_us": d.get("duration") * (1e-3 if d.get("duration_unit") == "ns" else
                                                    1e3 if d.get("duration_unit") == "ms" else 1),
               "issue_active_pct": d.get("issue_active_pct"), "fma_pipe_pct": d.get("fma_pipe_pct"),
               "occupancy_pct": d.get("occupancy_pct"), "registers": d.get("registers")}
        if fam == "blend":
            ent["pairs"] = work["fwd_pairs"]
        elif fam == "bwd_pixels":
            ent["pairs"] = work["bwd_pairs"]
        out[fam] = ent
    path = os.path.join(ROOT, "profiles", "ncu_kernels.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
