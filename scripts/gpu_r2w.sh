# diagnostics: C5 per-height trace, C2 PLU core sizes, C5 launch list
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
MFH_HEIGHT_TRACE=1 timeout 600 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c5_trace.log 2>&1; echo "c5 trace rc=$?"
MFH_HEIGHT_TRACE=1 MFH_PLU_TRACE=1 timeout 300 python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c2_trace.log 2>&1; echo "c2 trace rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --config c5 --profile --no-cpu-baseline > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
python scripts/summarize_launches.py gpurun_out/launches_c5.csv gpurun_out/launches_c5.txt > /dev/null
