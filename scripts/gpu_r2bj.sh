#!/bin/bash
# blocked-LU look-ahead: GPU suite, then same-box A/B at C5, C3, C4, C2
set -u
O=gpurun_out/bj; mkdir -p $O
export PYTHONFAULTHANDLER=1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for c in c5 c3 c4 c2; do
  for r in on off; do
    if [ $r = on ]; then unset MFH_LU_LOOKAHEAD_MIN; else export MFH_LU_LOOKAHEAD_MIN=100000000; fi
    timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_${c}_$r.log 2>&1; echo "bench $c lookahead $r rc=$?"
    python - <<PY
import json
l=[x for x in open("$O/bench_${c}_$r.log") if x.startswith("{")]
d=json.loads(l[-1]); pr=d.get("phase_roofline",{})
print("$c lookahead $r", round(d["value"],4), {k:(round(v["ms"],1), round(v.get("frac",0),3)) for k,v in pr.items() if isinstance(v,dict) and "ms" in v and k in ("skeleton","hodlr_factor","eliminate","dense_front")})
PY
  done
done
