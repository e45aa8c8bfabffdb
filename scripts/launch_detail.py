"""Per-launch detail of an ncu launch list: the longest launches of the named kernels with grid sizes."""
import csv
import sys
from collections import defaultdict

path, names = sys.argv[1], sys.argv[2:]
rows = [l for l in open(path) if l.startswith('"')]
d = defaultdict(dict)
for r in csv.DictReader(rows):
    d[r["ID"]][r["Metric Name"]] = r["Metric Value"]
    d[r["ID"]]["k"] = r["Kernel Name"].split("(")[0].replace("void ", "")
for name in names:
    L = sorted(((float(v["gpu__time_duration.sum"].replace(",", "")) / 1e3, v.get("launch__grid_size"))
                for v in d.values() if name in v["k"]), reverse=True)
    print(name, len(L), "total %.1f ms" % (sum(a for a, _ in L) / 1e3), [(round(a), b) for a, b in L[:14]])
