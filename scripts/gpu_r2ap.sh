# densify on k_gemm: bitwise test; C2 A/B of the threshold
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_densify.py -m gpu -x -q -rA -p no:cacheprovider > gpurun_out/t_ap.log 2>&1; echo "densify test rc=$?"; tail -3 gpurun_out/t_ap.log
for T in 4096 1024 256; do
  MFH_DENSIFY_MIN=$T timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ap_c2_$T.log 2>&1
  python - $T <<'PY'
import json, sys
for l in open(f"gpurun_out/ap_c2_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("c2 densify", sys.argv[1], round(d["value"], 4), "its", d["gmres"]["iterations"], "res", d["gmres"]["final_rel_residual"], {k: round(v, 2) for k, v in d["factor"]["phases_ms"].items()})
PY
done
