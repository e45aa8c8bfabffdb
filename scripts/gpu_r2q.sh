mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_mf.py tests/test_gpu_gmres.py tests/test_config_parity.py tests/test_gpu_shard.py -m gpu -x -q -rA -p no:cacheprovider > gpurun_out/t_q.log 2>&1; echo "tests rc=$?"
for i in 1 2; do
MFH_PDL=0 timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_pdl0_$i.log 2>&1; echo "bench0 rc=$?"
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_pdl1_$i.log 2>&1; echo "bench1 rc=$?"
done
