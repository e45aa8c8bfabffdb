# hybrid GEMV (k_gemv2 for one vector, DMMA for several) + implicit-pivoting Gauss-Jordan
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 300 python -m pytest tests/test_gpu_gemv.py tests/test_gpu_kernels.py -x -q -rA -p no:cacheprovider > gpurun_out/t_ac1.log 2>&1; echo "gemv+kernels rc=$?"; tail -2 gpurun_out/t_ac1.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_ac.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_ac.log
timeout 300 python scripts/inv_bench.py > gpurun_out/inv_bench2.log 2>&1; echo "inv rc=$?"; head -7 gpurun_out/inv_bench2.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ac_c2.log 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --param n_c=8192 > gpurun_out/bench_ac_c5b.log 2>&1; echo "c5b rc=$?"
for f in c2 c5b; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/bench_ac_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"], 4), "factor", round(d["split_s"]["factor_s"], 4), "gmres", round(d["split_s"]["gmres_inner_s"], 4),
              "its", d["gmres"]["iterations"], "apply ms", round(d["apply"]["ms"], 3), {k: round(v, 2) for k, v in d["factor"]["phases_ms"].items()})
PY
done
