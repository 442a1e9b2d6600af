"""Per-CTA, per-step timeline of the fused NPB CG kernel (k_cg_tiled) on class C
(experiment build with -DLILAC_CTA_TRACE=1):

    python tools/build_variant.py tr -DLILAC_CTA_TRACE=1
    LILAC_B200_LIB=variants/tr/liblilac_b200.so python tools/cg_trace.py

Per CG step (averaged over the steps of one NPB outer iteration): when the
gate (previous step's p complete) passes, when slab 0 of p lands, the walk's
end (min / avg / max over CTAs), and the two grid barriers. Times in us from
the step's first CTA start.
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402

STEPS, CTAS = 32, 160
L = N.lib()
N.check(L.b200_init(0))
rp, ci, val = D.gen_npb(150000, 15, 110.0)
A = D.Matrix.csr(rp, ci, val)
cg = D.CG(A)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    cg.outer(110.0, 25, s)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (STEPS * CTAS * 8))()
assert L.b200_debug_cg_trace(buf, STEPS * CTAS * 8) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(STEPS, CTAS, 8).astype(np.int64)
grid = int((a[0, :, 0] > 0).sum())
a = a[:, :grid, :]
steps = int((a[:, 0, 0] > 0).sum())
rows = []
for it in range(1, min(steps, 25)):
    t = a[it]
    t0 = t[:, 0].min()
    r = (t - t0) / 1e3
    last = np.argmax(r[:, 3])  # the CTA whose walk ends last
    rows.append([r[:, 1].min(), r[:, 1].max(), r[:, 2].mean(), r[:, 2].max(), r[:, 3].min(), r[:, 3].mean(),
                 r[:, 3].max(), r[last, 6], r[last, 7], r[:, 7].max(), r[:, 4].max(), r[:, 5].max(), (a[it + 1, :, 0].min() - t0) / 1e3 if it + 1 < steps else np.nan])
m = np.nanmean(np.array(rows), axis=0)
names = ["gate min", "gate max", "slab0 avg", "slab0 max", "walk end min", "walk end avg", "walk end max",
         "last: y+pq done", "last: staged", "arrive1 max", "barrier1 max", "barrier2 max", "next step start"]
print(f"grid {grid}, steps traced {steps}; per step (mean over steps 1..{len(rows)}), us from the step's first CTA start:")
for n, v in zip(names, m):
    print(f"  {n:16s} {v:8.2f}")

# is a CTA's SpMV time systematic across steps (same CTA, same SM, same tile)?
w = (a[1:steps, :, 3] - a[1:steps, :, 2]).astype(np.float64) / 1e3  # walk: slab 0 landed -> walk end
c = np.corrcoef(w[::2].mean(axis=0), w[1::2].mean(axis=0))[0, 1]
print(f"per-CTA walk time, even vs odd steps: correlation {c:.2f}; CTA means min/avg/max "
      f"{w.mean(axis=0).min():.2f}/{w.mean():.2f}/{w.mean(axis=0).max():.2f} us; per-step spread (max-avg) "
      f"{(w.max(axis=1) - w.mean(axis=1)).mean():.2f} us")

# systematic by SM or by tile? launch A with CTA b on tile b, launch B with
# CTA b on tile (b + 37) % grid; compare per-SM and per-tile mean walk times
def launch_walk(rot):
    assert L.b200_debug_cg_rot(rot) == 0
    cg.outer(110.0, 25, s)
    torch.cuda.synchronize()
    assert L.b200_debug_cg_trace(buf, STEPS * CTAS * 8) == 0
    sm = (C.c_uint * CTAS)()
    assert L.b200_debug_cg_smid(sm, CTAS) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(STEPS, CTAS, 8).astype(np.int64)[1:25, :grid]
    wk = ((t[:, :, 3] - t[:, :, 2]) / 1e3).mean(axis=0)
    by_sm = {int(sm[b]): wk[b] for b in range(grid)}
    by_tile = {(b + rot) % grid: wk[b] for b in range(grid)}
    return by_sm, by_tile
sa, ta = launch_walk(0)
sb, tb = launch_walk(37)
assert L.b200_debug_cg_rot(0) == 0
ks = sorted(set(sa) & set(sb))
print(f"per-SM walk time, launch A vs B (tiles rotated by 37): correlation "
      f"{np.corrcoef([sa[k] for k in ks], [sb[k] for k in ks])[0, 1]:.2f}; per-tile: "
      f"{np.corrcoef([ta[k] for k in range(grid)], [tb[k] for k in range(grid)])[0, 1]:.2f}")

# what explains the per-tile part? tile rows (row starts) vs nnz (tiles are nnz-balanced)
nt = grid
nnz_total = int(rp[-1])
bnd = [0]
for g in range(1, nt):
    tgt = (nnz_total * g + nt - 1) // nt
    r = int(np.searchsorted(rp, tgt, side="left"))
    bnd.append(max(min(r, len(rp) - 1), bnd[-1]))
bnd.append(len(rp) - 1)
bnd = np.array(bnd)
rows_t = np.diff(bnd)
nnz_t = rp[bnd[1:]] - rp[bnd[:-1]]
tm = np.array([(ta[k] + tb[k]) / 2 for k in range(nt)])
print(f"per-tile walk time vs rows: corr {np.corrcoef(tm, rows_t)[0, 1]:.2f}; vs nnz: {np.corrcoef(tm, nnz_t)[0, 1]:.2f}; "
      f"rows min/max {rows_t.min()}/{rows_t.max()}, nnz min/max {nnz_t.min()}/{nnz_t.max()}; "
      f"walk by tile index (first/last 10): {np.round(tm[:10], 1)} ... {np.round(tm[-10:], 1)}")
