# PLU window per-class completion times at C2 (one step), with core sizes
mkdir -p gpurun_out
MFH_PLU_EVENTS=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c2_pluev.log 2>&1; echo "rc=$?"
grep -c "plu window" gpurun_out/c2_pluev.log
