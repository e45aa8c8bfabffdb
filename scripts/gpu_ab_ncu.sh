# launch lists (ncu gpu__time_duration) of one C2 factorization+solve, new and base builds
L=paper_1410_2697_b200
cp $L/libmfh.so /tmp/libmfh_new2.so
for v in new base; do
  if [ $v = base ]; then cp $L/libmfh_base.so $L/libmfh.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$v.csv python bench.py --profile --no-cpu-baseline > gpurun_out/ncu_$v.log 2>&1
  echo "ncu $v rc=$?"
done
cp /tmp/libmfh_new2.so $L/libmfh.so
