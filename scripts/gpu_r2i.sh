mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_mf.py -m gpu -x -q -rA -p no:cacheprovider > gpurun_out/t_i.log 2>&1; echo "tests rc=$?"
MFH_BENCH_EMULATE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_emul2.log 2>&1; echo "emul2 rc=$?"
