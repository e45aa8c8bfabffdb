# round 2, call D: bench C2 with the new rooflines, ncu traffic + full captures, sanitizers
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_etree_abi.py tests/test_bench_cpu.py -m "gpu or not gpu" -x -q -rA -p no:cacheprovider > gpurun_out/t_etree.log 2>&1; echo "etree tests rc=$?"
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_c2.csv python bench.py --config c2 --profile > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_plu_cluster3 -s 4 -c 1 -o gpurun_out/r2_plu_cluster3 python bench.py --config c2 --profile > gpurun_out/ncu_plu.log 2>&1; echo "ncu plu rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sample_rb -s 2 -c 1 -o gpurun_out/r2_sample_rb python bench.py --config c2 --profile > gpurun_out/ncu_srb.log 2>&1; echo "ncu sample_rb rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sample$ -s 20 -c 1 -o gpurun_out/r2_sample python bench.py --config c2 --profile > gpurun_out/ncu_s.log 2>&1; echo "ncu sample rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemv2 -s 30 -c 1 -o gpurun_out/r2_gemv2 python bench.py --config c2 --profile > gpurun_out/ncu_gemv.log 2>&1; echo "ncu gemv rc=$?"
timeout 900 compute-sanitizer --tool memcheck --leak-check no python __graft_entry__.py smoke > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"
timeout 900 compute-sanitizer --tool racecheck python __graft_entry__.py smoke > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"
timeout 900 compute-sanitizer --tool synccheck python __graft_entry__.py smoke > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"
