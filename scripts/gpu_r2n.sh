mkdir -p gpurun_out
rm -f gpurun_out/ab_plu.txt
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$name.log 2>&1
  python - "$name" >> gpurun_out/ab_plu.txt <<'PY'
import json, sys
name = sys.argv[1]
for l in open(f"gpurun_out/ab_{name}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(name, round(d["value"], 4), {k: round(v, 1) for k, v in d["factor"]["phases_ms"].items()})
PY
}
run base
run cg MFH_PLU_CL16_GRID=1
run cg16 MFH_PLU_CL16_GRID=1 MFH_PLU_MAXGROUPS=16
run cg24 MFH_PLU_CL16_GRID=1 MFH_PLU_MAXGROUPS=24
run mg16 MFH_PLU_MAXGROUPS=16
run mg4 MFH_PLU_MAXGROUPS=4
run base2
cat gpurun_out/ab_plu.txt
