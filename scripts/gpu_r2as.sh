# one-barrier cluster panel LU; densified lr accounting
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_mf.py tests/test_gpu_gemm.py -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_as.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_as.log
timeout 300 python scripts/inv_bench.py > gpurun_out/inv_bench3.log 2>&1; tail -4 gpurun_out/inv_bench3.log
timeout 600 python bench.py --config c5 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/as_c5.log 2>&1; echo "c5 rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/as_c2.log 2>&1; echo "c2 rc=$?"
for f in c5 c2; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/as_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        pr = d["phase_roofline"]
        print(sys.argv[1], round(d["value"], 4), "its", d["gmres"]["iterations"], {k: round(v, 1) for k, v in d["factor"]["phases_ms"].items()})
        print("   ", {k: (round(v["frac"], 3), round(v["achieved"], 1)) for k, v in pr.items() if isinstance(v, dict)})
PY
done
