"""Per-kernel-class DRAM traffic and time of one bench step from an ncu CSV.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/traffic.csv \
        python bench.py --config c2 --profile
    python scripts/ncu_traffic.py gpurun_out/traffic.csv profiles/r2_traffic_c2.json

ncu serialises launches and replays each one (cold caches): absolute times
are not bench numbers, the per-launch DRAM bytes are what bench.py reports as
roofline.traffic (summed read + write per launch of the class).
"""
import csv
import json
import sys
from collections import defaultdict

CLASSES = [("k_plu", ("k_plu",)), ("k_sample", ("k_sample",)), ("k_gemm", ("k_gemm",)),
           ("k_gemv", ("k_gemv",)), ("k_spmv", ("k_spmv",)), ("k_inv", ("k_inv", "k_getrf", "k_trinv", "k_laswp")),
           ("k_mgs", ("k_mgs", "k_dot", "k_finish", "k_axpy")), ("cublas", ("cutlass", "gemm", "Kernel"))]


def klass(name):
    for k, pre in CLASSES:
        if any(name.startswith(p) or p in name for p in pre):
            return k
    return "other"


def main(path, out):
    per = defaultdict(dict)
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        key = r["ID"]
        per[key]["name"] = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = (r.get("Metric Unit") or "").lower()
        m = r["Metric Name"]
        if m == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
            per[key]["us"] = v
        elif m.startswith("dram__bytes"):
            v *= {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(unit, 1)
            per[key]["dram"] = per[key].get("dram", 0.0) + v
    agg = defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_bytes": 0.0, "kernels": set()})
    for d in per.values():
        a = agg[klass(d["name"])]
        a["launches"] += 1
        a["us"] += d.get("us", 0.0)
        a["dram_bytes"] += d.get("dram", 0.0)
        a["kernels"].add(d["name"])
    res = {}
    tot = sum(a["us"] for a in agg.values()) or 1.0
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        res[k] = {"launches": a["launches"], "time_ms": a["us"] / 1e3, "share": a["us"] / tot,
                  "dram_bytes": a["dram_bytes"], "dram_bytes_per_launch": a["dram_bytes"] / max(1, a["launches"]),
                  "dram_gbs_under_ncu": a["dram_bytes"] / max(1e-9, a["us"] * 1e-6) / 1e9,
                  "kernels": sorted(a["kernels"])}
    res["_source"] = ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none over one bench.py --profile step (serialised, cold caches)")
    json.dump(res, open(out, "w"), indent=1)
    for k, v in res.items():
        if not k.startswith("_"):
            print(f"{k:10s} launches {v['launches']:6d} time {v['time_ms']:9.3f} ms share {100 * v['share']:5.1f}% "
                  f"DRAM {v['dram_bytes'] / 1e6:10.1f} MB ({v['dram_bytes_per_launch'] / 1e6:8.3f} MB/launch)")


if __name__ == "__main__":
    main(*sys.argv[1:])
