# round 2, call A: config-scale parity, GPU suites, C5 memory breakdown
mkdir -p gpurun_out
TEST_FILES="tests/test_config_parity.py tests/test_gpu_kernels.py tests/test_gpu_mf.py tests/test_gpu_gmres.py" TEST_TIMEOUT=900 PYTEST_TIMEOUT=600 SMOKE=1 bash scripts/gpu_round.sh
MFH_MEM_TRACE=1 timeout 900 python bench.py --config c5 --profile > gpurun_out/c5_mem.log 2>&1; echo "c5 mem rc=$?"
MFH_MEM_TRACE=1 timeout 300 python bench.py --config c2 --profile > gpurun_out/c2_mem.log 2>&1; echo "c2 mem rc=$?"
