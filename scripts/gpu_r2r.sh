mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -m gpu -x -q -rA -p no:cacheprovider > gpurun_out/t_r.log 2>&1; echo "gemm tests rc=$?"
MFH_PLU_EVENTS=1 MFH_BENCH_NO_CLOCKS=1 timeout 300 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c2_plu_events.log 2>&1; echo "plu events rc=$?"
