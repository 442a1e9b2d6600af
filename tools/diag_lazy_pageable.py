"""Why does the lazy write-back move more on plain numpy vectors than on
pinned page-aligned ones? One NPB class A outer iteration of the C host loop
per memory kind, with per-harness byte counters and the lazy counters."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_07938_b200 import build as B  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402
from paper_2001_07938_b200 import harness as H  # noqa: E402

na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES["A"]
rp, ci, val = D.gen_npb(na, nonzer, shift)
E = C.CDLL(B.EX_LIB)
fn = E.npb_host_cg_outer
fn.restype = C.c_double
fn.argtypes = [C.c_int64] + [C.c_void_p] * 9 + [C.c_double, C.POINTER(C.c_double)]
H.set_writeback("lazy")
keep = []
for kind in sys.argv[1:] or ["pinned", "pageable"]:
    def vec(k):
        if kind == "pageable":
            a = np.zeros(k)
            keep.append(a)
            return a
        t = torch.zeros(k + 512, dtype=torch.float64, pin_memory=True)
        keep.append(t)
        a = t.numpy()
        off = (-a.ctypes.data % 4096) // 8
        return a[off:off + k]
    vs = [vec(na) for _ in range(6)]
    print(kind, [hex(v.ctypes.data) for v in vs], flush=True)
    x = vs[0]
    args = [na, rp.ctypes.data, val.ctypes.data, ci.ctypes.data] + [v.ctypes.data for v in vs]
    x[:] = 1.0
    rn = C.c_double()
    fn(*args, shift, C.byref(rn))
    x[:] = 1.0
    fn(*args, shift, C.byref(rn))
    s0, l0 = H.harness_stats(), H.lazy_counters()
    fn(*args, shift, C.byref(rn))
    s1, l1 = H.harness_stats(), H.lazy_counters()
    d = {k: {f: s1[k][f] - s0.get(k, {}).get(f, 0) for f in ("calls", "bytes_h2d", "bytes_d2h", "bytes_d2d")}
         for k in s1}
    print(kind, json.dumps(d), json.dumps({k: l1[k] - l0[k] for k in l1}), flush=True)
    H.host_sync()
    H.host_forget()
