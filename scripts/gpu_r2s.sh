mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_kernels.py tests/test_gpu_mf.py tests/test_config_parity.py tests/test_gpu_shard.py -m gpu -x -q -rA -p no:cacheprovider > gpurun_out/t_s.log 2>&1; echo "tests rc=$?"
for i in 1 2; do timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_s$i.log 2>&1; echo "bench rc=$?"; done
MFH_PLU_EVENTS=1 MFH_BENCH_NO_CLOCKS=1 timeout 300 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c2_plu_events.log 2>&1; echo "plu events rc=$?"
