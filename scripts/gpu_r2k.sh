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
run g96 MFH_PLU_GRID=96
run g64 MFH_PLU_GRID=64
run g48 MFH_PLU_GRID=48
run g96f MFH_PLU_GRID=96 MFH_PLU_COOP_FIRST=1
run g64f MFH_PLU_GRID=64 MFH_PLU_COOP_FIRST=1
run g48f MFH_PLU_GRID=48 MFH_PLU_COOP_FIRST=1
cat gpurun_out/ab_plu.txt
