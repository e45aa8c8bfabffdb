# densify default 256: whole suite, C1/C3/C4/C5 bench
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_aq.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_aq.log
for c in c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/aq_$c.log 2>&1; echo "$c rc=$?"
  python - $c <<'PY'
import json, sys
for l in open(f"gpurun_out/aq_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"], 4), "its", d["gmres"]["iterations"], "GB", round(d["factor"]["device_bytes"] / 1e9, 1), {k: round(v, 1) for k, v in d["factor"]["phases_ms"].items()})
PY
done
