mkdir -p gpurun_out
MFH_HEIGHT_TRACE=1 MFH_PLU_TRACE=1 MFH_BENCH_NO_CLOCKS=1 timeout 300 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c2_warm_trace.log 2>&1; echo "trace rc=$?"
