# grouped sampler tile order: tests, C5 + C2 bench
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_mf.py tests/test_config_parity.py tests/test_gpu_shard.py -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_am.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_am.log
timeout 600 python bench.py --config c5 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/am_c5.log 2>&1; echo "c5 rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/am_c2.log 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config c3 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/am_c3.log 2>&1; echo "c3 rc=$?"
for f in c5 c2 c3; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/am_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"], 4), "its", d["gmres"]["iterations"], {k: round(v, 1) for k, v in d["factor"]["phases_ms"].items()})
PY
done
