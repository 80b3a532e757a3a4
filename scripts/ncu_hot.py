"""Hot SASS / source lines of one kernel in an ncu report (run here).

    python scripts/ncu_hot.py gpurun_out/prof_k_blend.ncu-rep [--source cuda|sass] [--top 40]
"""
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    view = sys.argv[sys.argv.index("--source") + 1] if "--source" in sys.argv else "sass"
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    ic = hdr.index("Instructions Executed")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    src = hdr.index("Source")
    data = []
    total_i = total_s = 0
    for r in rows[1:]:
        try:
            n = float(r[ic] or 0)
            s = float(r[st] or 0)
        except (ValueError, IndexError):
            continue
        total_i += n
        total_s += s
        data.append((n, s, r[0], r[src].strip()))
    print(f"total warp instructions {total_i:.3e}, stall samples {total_s:.0f}")
    key = 1 if "--by-stall" in sys.argv else 0
    for n, s, addr, text in sorted(data, key=lambda x: -x[key])[:top]:
        print(f"{n:12.0f} {100 * n / max(total_i, 1):5.1f}%  stall {100 * s / max(total_s, 1):5.1f}%  {addr}  {text[:110]}")


if __name__ == "__main__":
    main()
