#!/bin/bash
# k_gemm_big against the cuBLAS route: GPU suite, then same-box A/B bench lines at C5, C3, C2
set -u
O=gpurun_out/bg; mkdir -p $O
export PYTHONFAULTHANDLER=1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.log
for c in c5 c3 c2; do
  for r in big blas; do
    MFH_GEMM_ROUTE=$r timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_${c}_$r.log 2>&1; echo "bench $c $r rc=$?"
    python - <<PY
import json
l=[x for x in open("$O/bench_${c}_$r.log") if x.startswith("{")]
d=json.loads(l[-1]); pr=d.get("phase_roofline",{})
print("$c $r", round(d["value"],4), {k:(round(v["ms"],1), round(v.get("frac",0),3)) for k,v in pr.items() if isinstance(v,dict) and "ms" in v})
PY
  done
done
