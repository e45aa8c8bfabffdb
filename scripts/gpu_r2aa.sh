# apply launch list at C2 (new GEMV) and ncu --set full of one k_inv_reg<16,4> (n = 128)
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
MFH_APPLY_TRACE=1 timeout 300 python scripts/apply_profile.py > gpurun_out/apply_prof.log 2>&1; echo "apply prof rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/apply_launches.csv python scripts/apply_profile.py > gpurun_out/ncu_apply.log 2>&1; echo "ncu apply rc=$?"
python scripts/summarize_launches.py gpurun_out/apply_launches.csv gpurun_out/apply_launches.txt > /dev/null
cat > /tmp/inv1.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1410_2697_b200 as P
from paper_1410_2697_b200 import _lib
n = 128
rng = np.random.default_rng(0)
blk = rng.standard_normal((n, n)) + 2 * n * np.eye(n)
for _ in range(3):
    buf = np.ascontiguousarray(blk.ravel().copy())
    sing = np.zeros(1, dtype=np.int32)
    _lib.check(_lib.lib().mfh_test_inverse_batched(_lib.context().handle, 1, _lib.ptr(np.zeros(1, dtype=np.int64)),
               _lib.ptr(np.array([n], dtype=np.int64)), _lib.ptr(buf), buf.size, _lib.ptr(sing)))
print("ok")
PY
timeout 300 python /tmp/inv1.py > gpurun_out/inv1.log 2>&1; echo "inv1 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_inv_reg -c 1 -o gpurun_out/inv_reg128 -f python /tmp/inv1.py > gpurun_out/ncu_inv.log 2>&1; echo "ncu inv rc=$?"
ncu -i gpurun_out/inv_reg128.ncu-rep --page source --csv > gpurun_out/inv_reg128_source.csv 2>/dev/null; echo "src rc=$?"
ncu -i gpurun_out/inv_reg128.ncu-rep --page details --csv > gpurun_out/inv_reg128_details.csv 2>/dev/null; echo "det rc=$?"
