#!/bin/bash
set -u
O=gpurun_out/bc; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -p no:cacheprovider -k spmv > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
for R in 256 128 64; do for S in 2 3 4; do
  echo "R=$R STG=$S"; MFH_SPMV_R=$R MFH_SPMV_STG=$S timeout 300 python scripts/spmv_bench.py all 2>&1 | grep -v "^c2"
done; done > $O/sweep.txt 2>&1
echo "P64 R=256 STG=2" >> $O/sweep.txt; MFH_SPMV_P64=1 timeout 300 python scripts/spmv_bench.py 2>&1 | grep -v "^c2" >> $O/sweep.txt
cat $O/sweep.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmv_stream --launch-skip 250 -c 1 -o $O/spmv_stream -f python scripts/spmv_bench.py > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/spmv_stream.ncu-rep --page details --csv > $O/spmv_stream_details.csv 2>/dev/null
