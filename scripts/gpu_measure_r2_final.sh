#!/bin/bash
# Final round-2 measurement set (every capture after its command exited 0 without ncu):
# GPU suite, smoke, C2 bench line with the CPU baseline, the reference arm, launch list,
# bench lines for C1/C3/C4/C5 and conventional C5, SpMV table.
set -u
O=gpurun_out/m4; mkdir -p $O
export PYTHONFAULTHANDLER=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 180 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python scripts/spmv_bench.py all > $O/spmv.txt 2>&1; cat $O/spmv.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c2.log 2>&1; echo "c2 bench rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_c2_reference.log 2>&1; echo "c2 reference arm rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --profile --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
python scripts/summarize_launches.py $O/launches_c2.csv $O/launches_c2.txt > /dev/null
for c in c1 c3 c4 c5; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.log 2>&1; echo "bench $c rc=$?"
done
timeout 900 python bench.py --config c5 --mode conventional --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_conv.log 2>&1; echo "bench c5 conv rc=$?"
MFH_GEMM_ROUTE=big timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_nolib.log 2>&1; echo "bench c5 library-free rc=$?"
ls $O
