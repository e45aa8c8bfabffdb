mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_mf.py tests/test_gpu_gmres.py tests/test_config_parity.py -m gpu -x -q -rA -p no:cacheprovider > gpurun_out/t_p.log 2>&1; echo "tests rc=$?"
MFH_PDL=0 timeout 300 python scripts/apply_profile.py > gpurun_out/apply_pdl0.log 2>&1; echo "pdl0 rc=$?"
MFH_PDL=1 timeout 300 python scripts/apply_profile.py > gpurun_out/apply_pdl1.log 2>&1; echo "pdl1 rc=$?"
grep "apply graph" gpurun_out/apply_pdl0.log | tail -1
grep "apply graph" gpurun_out/apply_pdl1.log | tail -1
MFH_PDL=0 timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_pdl0.log 2>&1; echo "bench0 rc=$?"
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench1 rc=$?"
