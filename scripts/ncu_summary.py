"""Summarise ncu reports (run here, no GPU): key throughput / stall metrics per captured kernel.

    python scripts/ncu_summary.py gpurun_out/prof_*.ncu-rep [--json profiles/ncu_summary_r01.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "smsp__inst_executed.sum": "warp_instructions",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__warps_eligible.avg.per_cycle_active": "eligible_warps",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_sb",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio": "stall_branch",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math_throttle",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio": "stall_mio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio": "stall_lg",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio": "stall_no_instr",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio": "stall_not_selected",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else path}
        for i, h in enumerate(hdr):
            if h in KEYS:
                v = vals[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                d[KEYS[h]] = v
                d[KEYS[h] + "_unit"] = units[i]
        res.append(d)
    return res


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    jpath = None
    if "--json" in sys.argv:
        jpath = sys.argv[sys.argv.index("--json") + 1]
        args = [a for a in args if a != jpath]
    allr = {}
    for p in args:
        for d in summarise(p):
            name = d["kernel"].split("(")[0].split("<")[0]
            allr[name] = d
            keys = ["duration", "sm_throughput_pct", "issue_active_pct", "occupancy_pct", "registers", "dram_pct",
                    "dram_read", "dram_write", "warp_instructions", "fma_pipe_pct", "fp64_pipe_pct", "lsu_pipe_pct",
                    "eligible_warps", "stall_wait", "stall_short_sb", "stall_long_sb", "stall_barrier",
                    "stall_branch", "stall_mio", "stall_lg"]
            print(name + ": " + ", ".join(f"{k}={d.get(k)}{d.get(k + '_unit', '')}" for k in keys if k in d))
    if jpath:
        with open(jpath, "w") as f:
            json.dump(allr, f, indent=1)


if __name__ == "__main__":
    main()
