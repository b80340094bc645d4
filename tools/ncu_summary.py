"""Summarise an ncu launch list (gpu__time_duration.sum CSV) by kernel name."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                 "nsecond": 1e-3}.get(unit, 1e-3)
        rows.append((int(r["ID"]), r["Kernel Name"], v * scale))
    return rows


def main(path, first=0, last=None):
    rows = load(path)
    rows = [r for r in rows if r[0] >= first and (last is None or r[0] <= last)]
    agg = defaultdict(lambda: [0, 0.0])
    for _, name, us in rows:
        key = name.split("(")[0][:90]
        agg[key][0] += 1
        agg[key][1] += us
    total = sum(v[1] for v in agg.values())
    print(f"{'kernel':90s} {'count':>6s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:90s} {c:6d} {t:10.1f} {t / c:9.2f} {100 * t / total:5.1f}%")
    print(f"total {total:.1f} us over {len(rows)} launches")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], int(a[1]) if len(a) > 1 else 0, int(a[2]) if len(a) > 2 else None)
