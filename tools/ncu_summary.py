#!/usr/bin/env python
"""Per-kernel summary of an ncu --csv launch list (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum, launch__grid_size).

  python tools/ncu_summary.py launches.csv [--top N]

Kernels are grouped by (name, grid size); times are ncu's cold-cache,
serialised per-launch durations, so compare shares, not absolutes."""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 60
    rows = defaultdict(lambda: {})
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        key = r["ID"]
        d = rows[key]
        d["name"] = r["Kernel Name"]
        v = r["Metric Value"].replace(",", "")
        unit = r["Metric Unit"]
        m = r["Metric Name"]
        x = float(v) if v else 0.0
        if m == "gpu__time_duration.sum":
            x *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}.get(unit, 1.0)
            d["us"] = x
        elif m.startswith("dram__bytes"):
            x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
            d["bytes"] = d.get("bytes", 0.0) + x
        elif m == "launch__grid_size":
            d["grid"] = int(x)
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for d in rows.values():
        name = d["name"].replace("(anonymous namespace)::", "")
        name = name.split("(")[0] if name.startswith("void") is False else name.split("(")[0]
        k = (name, d.get("grid", 0))
        a = agg[k]
        a[0] += 1
        a[1] += d.get("us", 0.0)
        a[2] += d.get("bytes", 0.0)
    total = sum(a[1] for a in agg.values())
    print(f"launches {len(rows)}  total {total / 1e3:.2f} ms")
    for (name, grid), (n, us, by) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100 * us / total:5.1f}% {n:5d}x {us / n:9.1f} us {by / n / 1e6:10.1f} MB/launch "
              f"{by / us / 1e3 if us else 0:8.0f} GB/s  grid {grid:7d}  {name[:90]}")


if __name__ == "__main__":
    main()
