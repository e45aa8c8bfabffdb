mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_plu_groups -c 1 -o gpurun_out/plu_groups -f python scripts/plu_grid.py 1728 971 > gpurun_out/ncu_plug.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/plu_groups.ncu-rep --page source --csv --print-source sass > gpurun_out/plu_groups_sass.csv 2>/dev/null; echo "sass rc=$?"
ncu -i gpurun_out/plu_groups.ncu-rep --page source --csv --print-source cuda > gpurun_out/plu_groups_src.csv 2>/dev/null; echo "src rc=$?"
ncu -i gpurun_out/plu_groups.ncu-rep --page details --csv > gpurun_out/plu_groups_details.csv 2>/dev/null; echo "det rc=$?"
