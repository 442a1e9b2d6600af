import sys, os, zlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle_lib as O
from paper_2001_07938_b200 import _native as N, harness as H
H.set_errors_return(True)
rng = np.random.default_rng(zlib.crc32(b"long_rows"))
rows, cols = 40, 200000
lens = rng.integers(5000, 60000, rows).astype(np.int64)
rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
ci = rng.integers(0, cols, int(rp[-1])).astype(np.int64)
val = rng.uniform(-2, 2, int(rp[-1]))
x = rng.uniform(-2, 2, cols)
for k in (b"auto", b"split", b"merge", b"split"):
    N.lib().b200_set_kernel(k)
    y = np.full(rows, np.nan)
    H.spmv_csr(rows, y, rp, val, x, ci)
    print(k, float(np.abs(y - O.spmv_csr(rp, ci, val, x)).max()), flush=True)
print("ok")
