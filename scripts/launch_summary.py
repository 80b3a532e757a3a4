"""Summarise an ncu launch list (gpu__time_duration per launch) into per-kernel totals and shares.

    python scripts/launch_summary.py gpurun_out/launches.csv --steps 4 [--json profiles/x.json]

The list is cold-cache and serialised (ncu), so compare SHARES with bench.py's live CUDA-event
shares, not absolute times. `--steps` = renders (train steps) the profiled command ran.
"""
import csv
import io
import json
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        ns = float(r["Metric Value"].replace(",", ""))
        a = agg.setdefault(name, {"launches": 0, "total_us": 0.0})
        a["launches"] += 1
        a["total_us"] += ns / 1e3
    total = sum(a["total_us"] for a in agg.values())
    out = {"source": path, "steps": steps, "total_us": total, "kernels": {}}
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["total_us"]):
        out["kernels"][k] = {"launches": a["launches"], "total_us": round(a["total_us"], 2),
                             "us_per_step": round(a["total_us"] / steps, 2),
                             "share": round(a["total_us"] / total, 4)}
        print(f"{k:40s} {a['launches']:5d} launches {a['total_us'] / steps:9.1f} us/step  {a['total_us'] / total:6.1%}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
