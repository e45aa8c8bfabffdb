# re-entry check: whole GPU suite as the driver runs it, smoke, default bench line
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rA -p no:cacheprovider --durations=30 > gpurun_out/t_v.log 2>&1; echo "tests rc=$?"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_v.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_v.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/t_v.log
