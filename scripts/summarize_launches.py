"""Summarize an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import csv
import sys
from collections import defaultdict


def main(path, out=None):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        rows.append((r["Kernel Name"], v * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for k, us in rows:
        name = k.split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    lines = [f"launches: {len(rows)}  total kernel time: {tot / 1e3:.2f} ms (cold-cache, serialized)",
             f"{'kernel':60s} {'count':>7s} {'total ms':>10s} {'share':>7s} {'avg us':>9s}"]
    for name, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name[:60]:60s} {c:7d} {us / 1e3:10.3f} {100 * us / tot:6.1f}% {us / c:9.1f}")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
