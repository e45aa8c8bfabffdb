#!/bin/bash
# Re-entry check: whole GPU suite, smoke, C2 bench line, launch list.
set -u
O=gpurun_out/ba; mkdir -p $O
export PYTHONFAULTHANDLER=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest.log
timeout 180 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c2.log 2>&1; echo "bench rc=$?"
tail -1 $O/bench_c2.log | cut -c1-600
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --profile --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
python scripts/summarize_launches.py $O/launches_c2.csv $O/launches_c2.txt > /dev/null
