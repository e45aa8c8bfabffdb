#!/bin/bash
set -u
O=gpurun_out/cc; mkdir -p $O
export PYTHONFAULTHANDLER=1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for c in c5 c3 c4 c2 c1; do
  timeout 900 python bench.py --config $c --steps 4 --warmup 2 --no-cpu-baseline > $O/bench_$c.log 2>&1; echo "bench $c rc=$?"
  python - <<PY
import json
l=[x for x in open("$O/bench_$c.log") if x.startswith("{")]
d=json.loads(l[-1]); f=d["factor"]
print("$c", round(d["value"],4), "e2e", round(d["e2e"]["value"],4), "device_ms", round(f["device_ms"],1), "idle", round(f["phases_ms"]["idle_gap_ms"],1), "select_host", round(f["host_ms"]["host_select_ms"],1), "its", d["gmres"]["iterations"])
PY
done
