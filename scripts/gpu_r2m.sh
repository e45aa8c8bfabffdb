mkdir -p gpurun_out
MFH_OP_TRACE=1 CUDA_LAUNCH_BLOCKING=1 timeout 900 python bench.py --config c5 --profile > gpurun_out/c5_optrace.log 2>&1; echo "c5 optrace rc=$?"
MFH_HEIGHT_TRACE=1 timeout 900 python bench.py --config c5 --profile > gpurun_out/c5_htrace.log 2>&1; echo "c5 htrace rc=$?"
