# tests + C2 bench (no CPU baseline) + optional other configs, for A/B of a change
mkdir -p gpurun_out; rm -f gpurun_out/summary.txt
TEST_FILES="${TEST_FILES:-tests/test_gpu_kernels.py tests/test_gpu_mf.py tests/test_gpu_gmres.py tests/test_gpu_shard.py}" TEST_TIMEOUT=600 PYTEST_TIMEOUT=300 SMOKE=1 bash scripts/gpu_round.sh > /dev/null
for cfg in ${BENCH_CFGS:-c2}; do
  timeout 900 python bench.py --config $cfg --steps ${BENCH_STEPS:-5} --warmup 3 --no-cpu-baseline > gpurun_out/bench_$cfg.log 2>&1; echo "bench $cfg rc=$?" >> gpurun_out/summary.txt
done
cat gpurun_out/summary.txt
