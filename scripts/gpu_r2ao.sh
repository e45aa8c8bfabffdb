# MGS register kernel at C5 size, two row groups per warp in k_gemv_tc
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_gemv.py tests/test_gpu_gmres.py tests/test_gpu_mf.py -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_ao.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_ao.log
timeout 600 python bench.py --config c5 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/ao_c5.log 2>&1; echo "c5 rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ao_c2.log 2>&1; echo "c2 rc=$?"
for f in c5 c2; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/ao_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"], 4), "gmres", round(d["split_s"]["gmres_inner_s"], 4), "its", d["gmres"]["iterations"], {k: round(v, 1) for k, v in d["factor"]["phases_ms"].items()})
PY
done
