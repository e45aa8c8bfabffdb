#!/bin/bash
# One GPU call: build check, GPU tests (per-file, bounded), smoke, small bench.
set -u
mkdir -p gpurun_out; rm -f gpurun_out/summary.txt
export PYTHONFAULTHANDLER=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/gpu.txt 2>&1
for f in ${TEST_FILES:-tests/test_gpu_kernels.py tests/test_gpu_mf.py tests/test_gpu_gmres.py}; do
  b=$(basename $f .py)
  timeout ${TEST_TIMEOUT:-300} python -m pytest $f -m gpu -v -x -rA -p no:cacheprovider ${PYTEST_EXTRA:-} --timeout ${PYTEST_TIMEOUT:-120} > gpurun_out/$b.log 2>&1
  echo "$b rc=$?" >> gpurun_out/summary.txt
done
if [ -n "${SMOKE:-1}" ]; then
  timeout 180 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
fi
for cfg in ${BENCH_CFGS:-}; do
  timeout ${BENCH_TIMEOUT:-300} python bench.py --config $cfg --steps ${BENCH_STEPS:-2} --warmup ${BENCH_WARMUP:-1} --no-cpu-baseline > gpurun_out/bench_$cfg.log 2>&1
  echo "bench $cfg rc=$?" >> gpurun_out/summary.txt
done
cat gpurun_out/summary.txt
