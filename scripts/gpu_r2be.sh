#!/bin/bash
set -u
O=gpurun_out/be; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -p no:cacheprovider -k spmv > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python scripts/spmv_bench.py all > $O/spmv_stream.txt 2>&1; cat $O/spmv_stream.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmv_stream --launch-skip 250 -c 1 -o $O/spmv_stream -f python scripts/spmv_bench.py > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/spmv_stream.ncu-rep --page details --csv > $O/spmv_stream_details.csv 2>/dev/null
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv python bench.py --config c5 --profile --no-cpu-baseline > $O/ncu_launch_c5.log 2>&1; echo "c5 launch list rc=$?"
python scripts/summarize_launches.py $O/launches_c5.csv $O/launches_c5.txt > /dev/null
head -45 $O/launches_c5.txt
