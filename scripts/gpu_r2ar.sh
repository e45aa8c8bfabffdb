# single-matrix Gauss-Jordan (n = 128): ncu --set full with SASS stalls
mkdir -p gpurun_out
cat > /tmp/inv1.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1410_2697_b200 as P
from paper_1410_2697_b200 import _lib
n = int(sys.argv[1])
rng = np.random.default_rng(0)
blk = rng.standard_normal((n, n)) + 2 * n * np.eye(n)
for _ in range(3):
    buf = np.ascontiguousarray(blk.ravel().copy())
    sing = np.zeros(1, dtype=np.int32)
    _lib.check(_lib.lib().mfh_test_inverse_batched(_lib.context().handle, 1, _lib.ptr(np.zeros(1, dtype=np.int64)),
               _lib.ptr(np.array([n], dtype=np.int64)), _lib.ptr(buf), buf.size, _lib.ptr(sing)))
print("ok")
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_inv_reg -s 2 -c 1 -o gpurun_out/inv128b -f python /tmp/inv1.py 128 > gpurun_out/ncu_inv128b.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/inv128b.ncu-rep --page source --csv --print-source sass > gpurun_out/inv128b_sass.csv 2>/dev/null; echo "sass rc=$?"
ncu -i gpurun_out/inv128b.ncu-rep --page raw --csv > gpurun_out/inv128b_raw.csv 2>/dev/null; echo "raw rc=$?"
