mkdir -p gpurun_out; rm -f gpurun_out/plu_grid.txt
for G in 148 74 49 37 25; do
  for s in "1728 971" "864 864"; do
    MFH_PLU_GRID=$G timeout 120 python scripts/plu_grid.py $s >> gpurun_out/plu_grid.txt 2>&1
  done
done
cat gpurun_out/plu_grid.txt
