mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_densify.py tests/test_gpu_mf.py tests/test_config_parity.py -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_au.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_au.log
MFH_HEIGHT_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c2_trace4.log 2>&1; echo "trace rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/au_c2.log 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config c5 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/au_c5.log 2>&1; echo "c5 rc=$?"
for f in c2 c5; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/au_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"], 4), "its", d["gmres"]["iterations"], {k: round(v, 1) for k, v in d["factor"]["phases_ms"].items()})
PY
done
