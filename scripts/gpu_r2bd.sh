#!/bin/bash
set -u
O=gpurun_out/bd; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -p no:cacheprovider -k spmv > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
for R in 256 128 64; do for S in 2 3 4; do
  echo "R=$R STG=$S"; MFH_SPMV_R=$R MFH_SPMV_STG=$S timeout 300 python scripts/spmv_bench.py all 2>&1 | grep -v "^c2"
done; done > $O/sweep.txt 2>&1
cat $O/sweep.txt
