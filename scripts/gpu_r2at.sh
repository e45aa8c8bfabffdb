mkdir -p gpurun_out
MFH_HEIGHT_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c2_trace3.log 2>&1; echo "rc=$?"
