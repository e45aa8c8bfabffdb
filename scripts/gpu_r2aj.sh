# row-parallel PLU sweep: PLU tests, per-step microbench, C2 bench
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_mf.py tests/test_config_parity.py -x -q -p no:cacheprovider > gpurun_out/t_aj.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_aj.log
rm -f gpurun_out/plu_grid4.txt
for G in 148 74; do for s in "1728 971" "864 864"; do MFH_PLU_FORCE3=1 MFH_PLU_GRID=$G timeout 120 python scripts/plu_grid.py $s | sed 's/^/groups3 /' >> gpurun_out/plu_grid4.txt 2>&1; done; done
cat gpurun_out/plu_grid4.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_aj_c2.log 2>&1; echo "c2 rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/bench_aj_c2.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("c2", round(d["value"], 4), "gmres", round(d["split_s"]["gmres_inner_s"], 4), {k: round(v, 2) for k, v in d["factor"]["phases_ms"].items()})
PY
