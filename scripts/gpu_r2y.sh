# DMMA GEMV: whole GPU suite, C2 bench, C5 at (4096, 2) and (8192, 2)
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t_y.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_y.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_y_c2.log 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_y_c5.log 2>&1; echo "c5 rc=$?"
timeout 600 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --param n_c=8192 > gpurun_out/bench_y_c5b.log 2>&1; echo "c5b rc=$?"
for f in c2 c5 c5b; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/bench_y_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"], 4), "factor", round(d["split_s"]["factor_s"], 4), "gmres", round(d["split_s"]["gmres_inner_s"], 4),
              "its", d["gmres"]["iterations"], "apply ms", round(d["apply"]["ms"], 3), "apply frac", round(d["phase_roofline"]["apply"]["frac"], 3))
PY
done
