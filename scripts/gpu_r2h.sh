mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_mf.py tests/test_gpu_shard.py tests/test_gpu_gmres.py tests/test_config_parity.py -m gpu -x -q -rA -p no:cacheprovider > gpurun_out/t_h.log 2>&1; echo "tests rc=$?"
MFH_APPLY_OPS=1 MFH_APPLY_TRACE=1 timeout 300 python scripts/apply_profile.py > gpurun_out/apply_ops_c2.log 2>&1; echo "apply ops rc=$?"
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
