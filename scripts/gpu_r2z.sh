# DMMA GEMV (fixed) + register MGS: GEMV test first, whole GPU suite, inverse microbench, C2 + C5 bench, C2 op trace
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 300 python -m pytest tests/test_gpu_gemv.py -x -q -rA -p no:cacheprovider > gpurun_out/t_gemv.log 2>&1; echo "gemv test rc=$?"; tail -3 gpurun_out/t_gemv.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_z.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_z.log
timeout 300 python scripts/inv_bench.py > gpurun_out/inv_bench.log 2>&1; echo "inv rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_z_c2.log 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --param n_c=8192 > gpurun_out/bench_z_c5b.log 2>&1; echo "c5b rc=$?"
for f in c2 c5b; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/bench_z_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"], 4), "factor", round(d["split_s"]["factor_s"], 4), "gmres", round(d["split_s"]["gmres_inner_s"], 4),
              "its", d["gmres"]["iterations"], "apply ms", round(d["apply"]["ms"], 3), "apply frac", round(d["phase_roofline"]["apply"]["frac"], 3))
PY
done
