# round 2 measurement set: every config's bench line, the C2 launch list / traffic, conventional C5
mkdir -p gpurun_out
for cfg in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/r2_bench_$cfg.log 2>&1; echo "bench $cfg rc=$?"
done
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c5.log 2>&1; echo "bench c5 rc=$?"
timeout 1500 python bench.py --config c5 --mode conventional --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c5_conv.log 2>&1; echo "bench c5 conv rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_c2.csv python bench.py --config c2 --profile > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
