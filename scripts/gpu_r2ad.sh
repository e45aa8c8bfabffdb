# full GPU suite; C5 n_c sweep on the current code; conventional C5
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/t_ad.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_ad.log
rm -f gpurun_out/sweep_ad.txt
for p in "8192 2" "12288 2" "16384 2" "8192 3"; do
  set -- $p
  timeout 400 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --param n_c=$1 --param d=$2 > gpurun_out/sw2_$1_$2.log 2>&1
  python - $1 $2 >> gpurun_out/sweep_ad.txt <<'PY'
import json, sys
a, b = sys.argv[1:]
ok = False
for l in open(f"gpurun_out/sw2_{a}_{b}.log"):
    if l.startswith("{"):
        d = json.loads(l); ok = True
        f = d["factor"]
        print(a, b, round(d["value"], 3), "factor", round(d["split_s"]["factor_s"], 3), "gmres", round(d["split_s"]["gmres_inner_s"], 3),
              "its", d["gmres"]["iterations"], d["gmres"]["converged"], "mem GB", round(f["device_bytes"] / 1e9, 1), "peak reals", f["peak_stored_reals"],
              {k: round(v) for k, v in f["phases_ms"].items()})
if not ok:
    print(a, b, "FAILED")
PY
done
timeout 600 python bench.py --config c5 --mode conventional --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c5_conv.log 2>&1; echo "conv rc=$?"
python - >> gpurun_out/sweep_ad.txt <<'PY'
import json
for l in open("gpurun_out/c5_conv.log"):
    if l.startswith("{"):
        d = json.loads(l); f = d["factor"]
        print("conv", round(d["value"], 3), "factor", round(d["split_s"]["factor_s"], 3), "gmres", round(d["split_s"]["gmres_inner_s"], 3), "mem GB", round(f["device_bytes"] / 1e9, 1), "peak reals", f["peak_stored_reals"])
PY
cat gpurun_out/sweep_ad.txt
