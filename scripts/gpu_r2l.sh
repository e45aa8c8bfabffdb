mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_config_parity.py tests/test_gpu_mf.py tests/test_gpu_shard.py -m gpu -x -q -rA -p no:cacheprovider > gpurun_out/t_l.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "bench c5 rc=$?"
