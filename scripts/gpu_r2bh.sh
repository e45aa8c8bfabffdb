#!/bin/bash
# hybrid GEMM routing against cuBLAS-only and k_gemm_big-only: same-box A/B bench lines at C5, C3
set -u
O=gpurun_out/bh; mkdir -p $O
export PYTHONFAULTHANDLER=1
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_densify.py -m gpu -x -q -p no:cacheprovider --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for c in c5 c3; do
  for r in hybrid blas big; do
    if [ $r = hybrid ]; then unset MFH_GEMM_ROUTE; else export MFH_GEMM_ROUTE=$r; fi
    timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_${c}_$r.log 2>&1; echo "bench $c $r rc=$?"
    python - <<PY
import json
l=[x for x in open("$O/bench_${c}_$r.log") if x.startswith("{")]
d=json.loads(l[-1]); pr=d.get("phase_roofline",{})
print("$c $r", round(d["value"],4), {k:(round(v["ms"],1), round(v.get("frac",0),3)) for k,v in pr.items() if isinstance(v,dict) and "ms" in v and k in ("skeleton","hodlr_factor","eliminate","dense_front","sample")})
PY
  done
done
unset MFH_GEMM_ROUTE
for m in 1073741824 4294967296 8589934592; do
  MFH_GEMM_BLAS_MIN=$m timeout 900 python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_c5_min$m.log 2>&1
  python - <<PY
import json
l=[x for x in open("$O/bench_c5_min$m.log") if x.startswith("{")]
d=json.loads(l[-1]); print("c5 blas_min $m", round(d["value"],4))
PY
done
