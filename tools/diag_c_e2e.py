"""C host-loop e2e (examples/npb_host_cg.c) vs the Python loop, per write-back
mode, with the marshal runtime's fault / mprotect / hash counters."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402

N.check(N.lib().b200_init(0))
na, nonzer, niter, shift, _ = bench.NPB[sys.argv[1] if len(sys.argv) > 1 else "C"]
rp, ci, val = D.gen_npb(na, nonzer, shift)


def mc():
    a = np.zeros(4, np.int64)
    N.lib().b200_marshal_counters(N.ptr(a[0:1]), N.ptr(a[1:2]), N.ptr(a[2:3]), N.ptr(a[3:4]))
    return a.copy()


for name, fn in (("C", bench.e2e_c_host_cg), ("python", bench.e2e_harness_cg)):
    for mode in ("eager", "lazy"):
        m0 = mc()
        r = fn(rp, ci, val, na, shift, 3, mode)
        d = mc() - m0
        print(f"{name:6s} {mode:5s} {r['value']:8.1f} it/s  faults={d[0]} mprotects={d[1]} hashed={d[2]}", flush=True)
