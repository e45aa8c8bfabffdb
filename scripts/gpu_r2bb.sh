#!/bin/bash
set -u
O=gpurun_out/bb; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -p no:cacheprovider -k spmv > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
timeout 600 python scripts/spmv_bench.py all > $O/spmv_stream.txt 2>&1; cat $O/spmv_stream.txt
MFH_SPMV_NO_STREAM=1 timeout 600 python scripts/spmv_bench.py all > $O/spmv_old.txt 2>&1; cat $O/spmv_old.txt
