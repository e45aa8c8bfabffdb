#!/bin/bash
set -u
O=gpurun_out/bo; mkdir -p $O
export PYTHONFAULTHANDLER=1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 200 python scripts/spmv_bench.py all > $O/spmv.txt 2>&1; cat $O/spmv.txt
for c in c2 c5 c3; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_$c.log 2>&1; echo "bench $c rc=$?"
  python - <<PY
import json
l=[x for x in open("$O/bench_$c.log") if x.startswith("{")]
d=json.loads(l[-1]); pr=d.get("phase_roofline",{})
print("$c", round(d["value"],4), {k:(round(v["ms"],1), round(v.get("frac",0),3)) for k,v in pr.items() if isinstance(v,dict) and "ms" in v})
PY
done
