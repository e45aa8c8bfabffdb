"""Print an ncu launch list (gpu__time_duration.sum [+ grid, dram read]) in launch order."""
import csv
import sys

rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
d, order = {}, []
for r in csv.DictReader(rows):
    if r["ID"] not in d:
        order.append(r["ID"])
        d[r["ID"]] = {}
    d[r["ID"]][r["Metric Name"]] = r["Metric Value"]
    d[r["ID"]]["k"] = r["Kernel Name"].split("(")[0].replace("void ", "")[:34]
tot = 0.0
for i in order:
    v = d[i]
    t = float(v["gpu__time_duration.sum"].replace(",", "")) / 1e3
    tot += t
    rd = v.get("dram__bytes_read.sum")
    rd = "%8.2f MB" % (float(rd.replace(",", "")) / 1e6) if rd else ""
    print(f'{v["k"]:34s} {t:8.2f} us grid {v.get("launch__grid_size", ""):>6} {rd}')
print("total %.1f us" % tot)
