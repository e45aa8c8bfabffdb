mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_shard.py -m gpu -x -q -rA -p no:cacheprovider > gpurun_out/t_o.log 2>&1; echo "tests rc=$?"
