# GEMV v3 (64-column passes, 128-column segments): GEMV test, apply-related tests, apply launch list, C2 + C5 bench
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 300 python -m pytest tests/test_gpu_gemv.py -x -q -rA -p no:cacheprovider > gpurun_out/t_gemv.log 2>&1; echo "gemv test rc=$?"; tail -2 gpurun_out/t_gemv.log
timeout 900 python -m pytest tests/test_gpu_mf.py tests/test_gpu_gmres.py tests/test_gpu_shard.py tests/test_config_parity.py -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_ab.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_ab.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/apply_launches.csv python scripts/apply_profile.py > gpurun_out/ncu_apply.log 2>&1; echo "ncu apply rc=$?"
python scripts/summarize_launches.py gpurun_out/apply_launches.csv gpurun_out/apply_launches.txt | head -8
grep "apply graph replay" gpurun_out/ncu_apply.log | tail -1
timeout 300 python scripts/apply_profile.py 2>&1 | grep "replay\|host-array"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ab_c2.log 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --param n_c=8192 > gpurun_out/bench_ab_c5b.log 2>&1; echo "c5b rc=$?"
for f in c2 c5b; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/bench_ab_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(sys.argv[1], round(d["value"], 4), "factor", round(d["split_s"]["factor_s"], 4), "gmres", round(d["split_s"]["gmres_inner_s"], 4),
              "its", d["gmres"]["iterations"], "apply ms", round(d["apply"]["ms"], 3), "apply frac", round(d["phase_roofline"]["apply"]["frac"], 3))
PY
done
