# C5 at n_c 12288: height trace (host decide), PLU core sizes, launch list
mkdir -p gpurun_out
MFH_HEIGHT_TRACE=1 MFH_PLU_TRACE=1 MFH_INV_LOG=1 timeout 600 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c5b_trace.log 2>&1; echo "c5 trace rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5b.csv python bench.py --config c5 --profile --no-cpu-baseline > gpurun_out/ncu_c5b.log 2>&1; echo "ncu c5 rc=$?"
python scripts/summarize_launches.py gpurun_out/launches_c5b.csv gpurun_out/launches_c5b.txt > /dev/null
head -25 gpurun_out/launches_c5b.txt
