TEST_FILES="tests/test_gpu_kernels.py tests/test_gpu_mf.py tests/test_gpu_gmres.py tests/test_gpu_shard.py" TEST_TIMEOUT=600 PYTEST_TIMEOUT=300 bash scripts/gpu_round.sh
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.log 2>&1; echo "bench default rc=$?" >> gpurun_out/summary.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --profile --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
