mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_baseline_precond.py tests/test_etree_abi.py tests/test_gpu_gmres.py -m gpu -x -q -rA -p no:cacheprovider > gpurun_out/t_precond.log 2>&1; echo "precond tests rc=$?"
MFH_HEIGHT_TRACE=1 MFH_PLU_TRACE=1 timeout 300 python bench.py --config c2 --profile > gpurun_out/c2_height_trace.log 2>&1; echo "trace rc=$?"
