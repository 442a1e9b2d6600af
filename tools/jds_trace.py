"""Per-block timeline of k_jds on the Parboil shape (experiment build with
-DLILAC_CTA_TRACE=1): block entry / exit spread, waves, and exit time by the
block's longest jagged row.

    python tools/build_variant.py tr -DLILAC_CTA_TRACE=1
    LILAC_B200_LIB=variants/tr/liblilac_b200.so python tools/jds_trace.py
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402
from paper_2001_07938_b200 import workloads as W  # noqa: E402

L = N.lib()
N.check(L.b200_init(0))
rp, ci, val = W.gen_parboil()
perm, nzcnt, jd_ptr, jval, jcol = W.csr_to_jds(rp, ci, val)
A = D.Matrix.jds(nzcnt, perm, jval, jd_ptr, jcol)
n = len(rp) - 1
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
for _ in range(20):
    A.spmv(x.data_ptr(), y.data_ptr(), s)
torch.cuda.synchronize()
if not hasattr(L, "b200_debug_jds_trace"):  # a product build: the launches above are the workload (ncu)
    print("no trace in this build (-DLILAC_CTA_TRACE=1)")
    sys.exit(0)
buf = (C.c_ulonglong * (3 * 4096))()
assert L.b200_debug_jds_trace(buf, 3 * 4096) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 3).astype(np.int64)
a = a[a[:, 1] > 0]
nb = len(a)
t0 = a[:, 1].min()
ent, ex = (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3
life = ex - ent
print(f"blocks {nb}; entry: max {ent.max():.2f} us, exit: max {ex.max():.2f} us")
print(f"block lifetime min/avg/max {life.min():.2f}/{life.mean():.2f}/{life.max():.2f} us")
late = ent > 1.0
print(f"blocks entering after 1 us (second wave): {late.sum()}, their entry min {ent[late].min() if late.any() else 0:.2f}")
order = np.argsort(ex)
print("exit time quantiles (us):", " ".join(f"{q}:{np.quantile(ex, q):.2f}" for q in (0.1, 0.5, 0.9, 0.99, 1.0)))
print("entry time quantiles (us):", " ".join(f"{q}:{np.quantile(ent, q):.2f}" for q in (0.1, 0.5, 0.9, 0.99, 1.0)))
