#!/bin/bash
set -u
O=gpurun_out/bt; mkdir -p $O
export PYTHONFAULTHANDLER=1
for c in c2 c3 c4 c5 c1; do
  for t in default 1; do
    if [ $t = default ]; then unset MFH_PLAN_THREADS; else export MFH_PLAN_THREADS=$t; fi
    timeout 900 python bench.py --config $c --steps 4 --warmup 2 --no-cpu-baseline > $O/bench_${c}_$t.log 2>&1; echo "bench $c threads $t rc=$?"
    python - <<PY
import json
l=[x for x in open("$O/bench_${c}_$t.log") if x.startswith("{")]
d=json.loads(l[-1]); f=d["factor"]
print("$c plan threads $t", round(d["value"],4), "factor", round(d["split_s"]["factor_s"],4), "device_ms", round(f["device_ms"],1), "phases", round(sum(f["phases_ms"].values()),1), "its", d["gmres"]["iterations"])
PY
  done
done
