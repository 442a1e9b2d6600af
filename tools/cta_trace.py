"""Per-CTA timeline of the standalone tiled SpMV on NPB class C (experiment
build with -DLILAC_CTA_TRACE=1, see tools/build_variant.py):

    python tools/build_variant.py tr -DLILAC_CTA_TRACE=1
    LILAC_B200_LIB=variants/tr/liblilac_b200.so python tools/cta_trace.py

For three launches (each the last of 10 back-to-back ones): the spread of CTA
entry, first-slab arrival, walk end and exit across the grid, and how well
the per-SM walk time of one launch predicts the next (systematic per-SM speed
vs per-tile work).
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402

L = N.lib()
N.check(L.b200_init(0))
L.b200_set_kernel(b"tiled")
rp, ci, val = D.gen_npb(150000, 15, 110.0)
A = D.Matrix.csr(rp, ci, val)
x = torch.rand(150000, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
buf = (C.c_ulonglong * (5 * 1024))()
runs = []
for rep in range(3):
    for _ in range(10):
        A.spmv(x.data_ptr(), y.data_ptr(), s)
    torch.cuda.synchronize()
    assert L.b200_debug_cta_trace(buf, 5 * 1024) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 5)[:148].astype(np.int64).copy()
    runs.append(a)
    t0 = a[:, 1].min()
    ent, first, walk, ex = (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3, (a[:, 3] - t0) / 1e3, (a[:, 4] - t0) / 1e3
    print(f"launch {rep}: entry max {ent.max():.2f} us; first slab landed min/avg/max "
          f"{first.min():.2f}/{first.mean():.2f}/{first.max():.2f}; walk end min/avg/max "
          f"{walk.min():.2f}/{walk.mean():.2f}/{walk.max():.2f}; exit max {ex.max():.2f}")
    d = walk - first
    print(f"   walk duration min/avg/max {d.min():.2f}/{d.mean():.2f}/{d.max():.2f} us, std {d.std():.2f}")
# systematic per SM? correlate walk durations by SM id and by CTA (tile)
def dur_by(a, key):
    return {int(k): (v[3] - v[2]) / 1e3 for k, v in zip(a[:, 0] if key == "sm" else range(len(a)), a)}
for key in ("sm", "cta"):
    d0, d1 = dur_by(runs[0], key), dur_by(runs[1], key)
    ks = sorted(set(d0) & set(d1))
    c = np.corrcoef([d0[k] for k in ks], [d1[k] for k in ks])[0, 1]
    print(f"walk duration correlation across launches by {key}: {c:.2f} ({len(ks)} keys)")
a = runs[2]
order = np.argsort(a[:, 0])
dd = (a[order, 3] - a[order, 2]) / 1e3
print("walk duration by SM id (launch 2):", " ".join(f"{v:.1f}" for v in dd))
