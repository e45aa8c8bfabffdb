"""Key metrics of an `ncu --set full` capture (details page CSV) per launch:
duration, DRAM throughput and bytes, SM / tensor pipe utilisation, IPC,
occupancy, registers, warp-stall reasons.

    ncu -i rep.ncu-rep --page details --csv > details.csv
    python scripts/ncu_summary.py details.csv [out.txt]"""
import csv
import sys
from collections import OrderedDict

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "L2 Hit Rate", "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "No Eligible"]


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    launches = OrderedDict()
    for r in rows[1:]:
        if len(r) <= ix["Metric Value"]:
            continue
        key = (r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0].replace("void ", ""))
        name = r[ix["Metric Name"]]
        if name in KEYS:
            launches.setdefault(key, OrderedDict())[name] = f'{r[ix["Metric Value"]]} {r[ix["Metric Unit"]]}'.strip()
        if r[ix["Section Name"]] == "Warp State Statistics" and name.startswith("Stall"):
            launches.setdefault(key, OrderedDict())[name] = f'{r[ix["Metric Value"]]} {r[ix["Metric Unit"]]}'.strip()
    lines = []
    for (lid, kname), m in launches.items():
        lines.append(f"launch {lid}: {kname}")
        for k in KEYS:
            if k in m:
                lines.append(f"  {k:38s} {m[k]}")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
