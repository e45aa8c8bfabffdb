mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_kernels.py tests/test_gpu_mf.py tests/test_config_parity.py tests/test_gpu_shard.py -m gpu -x -q -rA -p no:cacheprovider > gpurun_out/t_u.log 2>&1; echo "tests rc=$?"
rm -f gpurun_out/ab_u.txt
for i in 1 2; do
 for v in prev new; do
  if [ $v = prev ]; then export MFH_LIB_VARIANT=prev; else unset MFH_LIB_VARIANT; fi
  timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_u_$v$i.log 2>&1
  python - $v$i >> gpurun_out/ab_u.txt <<'PY'
import json, sys
n = sys.argv[1]
for l in open(f"gpurun_out/ab_u_{n}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(n, round(d["value"], 4), {k: round(v, 1) for k, v in d["factor"]["phases_ms"].items()}, round(d["split_s"]["gmres_inner_s"], 4))
PY
 done
done
unset MFH_LIB_VARIANT
cat gpurun_out/ab_u.txt
