# densified large child updates: suite, C5 (+ MFH_DENSIFY_MIN=0 A/B, + MFH_DENSE_FRAC=0.3), C3, C2
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_an.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_an.log
timeout 600 python bench.py --config c5 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/an_c5.log 2>&1; echo "c5 rc=$?"
MFH_DENSE_FRAC=0.3 timeout 600 python bench.py --config c5 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/an_c5_df.log 2>&1; echo "c5 dense-frac rc=$?"
timeout 600 python bench.py --config c3 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/an_c3.log 2>&1; echo "c3 rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/an_c2.log 2>&1; echo "c2 rc=$?"
for f in c5 c5_df c3 c2; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/an_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"], 4), "its", d["gmres"]["iterations"], "res", d["gmres"]["final_rel_residual"], "GB", round(d["factor"]["device_bytes"] / 1e9, 1), {k: round(v, 1) for k, v in d["factor"]["phases_ms"].items()})
PY
done
