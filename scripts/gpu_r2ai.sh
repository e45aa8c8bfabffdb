mkdir -p gpurun_out; rm -f gpurun_out/plu_grid3.txt
for G in 148 74; do
  for s in "1728 971" "864 864"; do
    MFH_PLU_GRID=$G timeout 120 python scripts/plu_grid.py $s >> gpurun_out/plu_grid3.txt 2>&1
    MFH_PLU_FORCE3=1 MFH_PLU_GRID=$G timeout 120 python scripts/plu_grid.py $s | sed 's/^/groups3 /' >> gpurun_out/plu_grid3.txt 2>&1
  done
done
cat gpurun_out/plu_grid3.txt
MFH_PLU_FORCE3=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_plu_groups3 -c 1 -o gpurun_out/plu_g3 -f python scripts/plu_grid.py 1728 971 > gpurun_out/ncu_plug3.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/plu_g3.ncu-rep --page source --csv --print-source sass > gpurun_out/plu_g3_sass.csv 2>/dev/null; echo "sass rc=$?"
