# A/B of two builds on one box: paper_1410_2697_b200/libmfh.so (new) against
# paper_1410_2697_b200/libmfh_base.so (baseline), alternating, C2 bench lines.
set -u
mkdir -p gpurun_out
L=paper_1410_2697_b200
cp $L/libmfh.so /tmp/libmfh_new.so
: > gpurun_out/ab.txt
for r in 1 2; do
  for v in ${AB_VARIANTS:-new base}; do
    # variant "name" or "name:ENV=VAL" (env applied to the new build)
    vn=${v%%:*}; ve=""; case $v in *:*) ve=${v#*:};; esac
    if [ $vn = base ]; then cp $L/libmfh_base.so $L/libmfh.so; else cp /tmp/libmfh_new.so $L/libmfh.so; fi
    for cfg in ${AB_CFGS:-c2}; do
      env $ve timeout 900 python bench.py --config $cfg --steps ${AB_STEPS:-5} --warmup 3 --no-cpu-baseline > gpurun_out/ab_${vn}_${cfg}_$r.log 2>&1
      tail -1 gpurun_out/ab_${vn}_${cfg}_$r.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['factor']['phases_ms']
print('$vn $cfg r$r', round(d['value'],5), 'e2e', round(d['e2e']['value'],5), 'its', d['gmres']['iterations'], ' '.join('%s=%.2f'%(k[:-3],v) for k,v in p.items()))" >> gpurun_out/ab.txt 2>&1
    done
  done
done
cp /tmp/libmfh_new.so $L/libmfh.so
cat gpurun_out/ab.txt
