# batched descriptor transfers (skeleton / HODLR / eliminate / dense elimination): suite, C2 + C5 bench
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_ae.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_ae.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ae_c2.log 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --param n_c=12288 > gpurun_out/bench_ae_c5.log 2>&1; echo "c5 rc=$?"
for f in c2 c5; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/bench_ae_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"], 4), "factor", round(d["split_s"]["factor_s"], 4), "gmres", round(d["split_s"]["gmres_inner_s"], 4),
              "its", d["gmres"]["iterations"], "apply ms", round(d["apply"]["ms"], 3), {k: round(v, 2) for k, v in d["factor"]["phases_ms"].items()})
PY
done
