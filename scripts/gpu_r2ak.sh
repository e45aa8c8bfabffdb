# executed-flop rooflines, clock sampler, inverse sizes at C2, cuBLAS vs DMMA A/B at C5
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_ak.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_ak.log
timeout 300 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ak_c1.log 2>&1; echo "c1 rc=$?"; grep -o '"clocks": {[^}]*}' gpurun_out/ak_c1.log
MFH_INV_LOG=1 MFH_HEIGHT_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ak_c2_trace.log 2>&1; echo "c2 trace rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ak_c2.log 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config c5 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/ak_c5.log 2>&1; echo "c5 rc=$?"
MFH_GEMM_NO_BLAS=1 timeout 600 python bench.py --config c5 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/ak_c5_noblas.log 2>&1; echo "c5 noblas rc=$?"
for f in c2 c5 c5_noblas; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/ak_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        pr = d["phase_roofline"]
        print(sys.argv[1], round(d["value"], 4), {k: round(v, 1) for k, v in d["factor"]["phases_ms"].items()})
        print("   ", {k: (round(v["achieved"], 2), round(v["frac"], 3), round(v.get("ref_tflops") or 0, 2)) for k, v in pr.items() if isinstance(v, dict) and v.get("unit") == "TFLOP/s"})
PY
done
