# C5 (n_c, d) sweep, 1 timed step each
mkdir -p gpurun_out
rm -f gpurun_out/sweep_c5.txt
for p in "8192 2" "8192 1" "4096 1" "2048 2" "4096 3"; do
  set -- $p
  timeout 400 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --param n_c=$1 --param d=$2 > gpurun_out/sw_$1_$2.log 2>&1
  python - $1 $2 >> gpurun_out/sweep_c5.txt <<'PY'
import json, sys
a, b = sys.argv[1:]
ok = False
for l in open(f"gpurun_out/sw_{a}_{b}.log"):
    if l.startswith("{"):
        d = json.loads(l); ok = True
        f = d["factor"]
        print(a, b, round(d["value"], 3), "factor", round(d["split_s"]["factor_s"], 3), "gmres", round(d["split_s"]["gmres_inner_s"], 3),
              "its", d["gmres"]["iterations"], d["gmres"]["converged"], "mem GB", round(f["device_bytes"] / 1e9, 1),
              {k: round(v) for k, v in f["phases_ms"].items()})
if not ok:
    print(a, b, "FAILED")
PY
done
cat gpurun_out/sweep_c5.txt
