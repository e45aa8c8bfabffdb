# Round-2 measurement set (every capture after its command exited 0 without ncu):
# C2 bench line with CPU baseline, launch list, DRAM traffic per kernel class,
# ncu --set full of the new kernels, bench lines for C1/C3/C4/C5 and conventional C5.
set -u
mkdir -p gpurun_out/m3
O=gpurun_out/m3
export PYTHONFAULTHANDLER=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $O/gpu.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c2.log 2>&1; echo "c2 bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --profile --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
python scripts/summarize_launches.py $O/launches_c2.csv $O/launches_c2.txt > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/traffic_c2.csv python bench.py --profile --no-cpu-baseline > $O/ncu_traffic.log 2>&1; echo "traffic rc=$?"
python scripts/ncu_traffic.py $O/traffic_c2.csv $O/r2_traffic_c2.json > /dev/null; echo "traffic json rc=$?"
# --set full of the round-2 kernels: one-vector GEMV (C2 apply), Gauss-Jordan inverse, register MGS
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemv2 --launch-skip 200 -c 2 -o $O/gemv2 -f python bench.py --profile --no-cpu-baseline > $O/ncu_gemv2.log 2>&1; echo "ncu gemv2 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_inv_reg -c 2 -o $O/inv_reg -f python bench.py --profile --no-cpu-baseline > $O/ncu_inv.log 2>&1; echo "ncu inv rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mgs_reg -c 2 -o $O/mgs_reg -f python bench.py --profile --no-cpu-baseline > $O/ncu_mgs.log 2>&1; echo "ncu mgs rc=$?"
for r in gemv2 inv_reg mgs_reg; do ncu -i $O/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>/dev/null; done
# other configs (bounded CPU-baseline samples included)
for c in c1 c3 c4 c5; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.log 2>&1; echo "bench $c rc=$?"
done
timeout 900 python bench.py --config c5 --mode conventional --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_conv.log 2>&1; echo "bench c5 conv rc=$?"
# C5 batched GEMV under ncu (several right-hand sides, FP64 tensor cores)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemv_tc --launch-skip 40 -c 2 -o $O/gemv_tc -f python bench.py --config c5 --profile --no-cpu-baseline > $O/ncu_gemv_tc.log 2>&1; echo "ncu gemv_tc rc=$?"
ncu -i $O/gemv_tc.ncu-rep --page details --csv > $O/gemv_tc_details.csv 2>/dev/null
ls $O
