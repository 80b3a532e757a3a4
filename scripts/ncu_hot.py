"""Hot CUDA source lines (or SASS) of one kernel in an ncu report (run here, no GPU).

    python scripts/ncu_hot.py gpurun_out/prof_k_blend.ncu-rep [--sass] [--top 40]

Aggregates warp-stall samples and executed warp instructions per CUDA line (all files of the
kernel, inlined headers included) from the mixed cuda,sass source page.
"""
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    sass = "--sass" in sys.argv
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass" if sass else "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    data, fname, hdr = [], "", None
    tot_s = tot_i = 0.0
    for r in rows:
        if not r:
            continue
        if r[0] in ("File Name", "File Path"):
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Line No", "Address"):
            hdr = r
            continue
        if hdr is None or r[0] in ("Kernel Name", "Function Name"):
            continue
        try:
            si = hdr.index("Warp Stall Sampling (All Samples)")
            ii = hdr.index("Instructions Executed")
        except ValueError:
            continue
        if sass:
            key, src = r[0], r[1]
        else:
            if not r[0]:
                continue  # SASS row under a CUDA line
            key, src = f"{fname}:{r[0]}", r[1]
        try:
            s = float(r[si] or 0)
            n = float(r[ii] or 0)
        except ValueError:
            continue
        tot_s += s
        tot_i += n
        data.append((s, n, key, src.strip()))
    data.sort(reverse=True)
    print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
    for s, n, key, src in data[:top]:
        print(f"{100 * s / max(tot_s, 1):5.1f}% smp {100 * n / max(tot_i, 1):5.1f}% ins  {key:18s} {src[:110]}")


if __name__ == "__main__":
    main()
