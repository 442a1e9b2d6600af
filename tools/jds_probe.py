"""Parboil-shape JDS SpMV, back-to-back launches (for an ncu launch list)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402
from paper_2001_07938_b200 import workloads as W  # noqa: E402

N.check(N.lib().b200_init(0))
rp, ci, val = W.gen_parboil()
perm, nzcnt, jd_ptr, jval, jcol = W.csr_to_jds(rp, ci, val)
A = D.Matrix.jds(nzcnt, perm, jval, jd_ptr, jcol)
n = len(perm)
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for _ in range(reps):
    A.spmv(x.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(20_000_000)  # hold the stream until all 200 launches are queued
e0.record()
for _ in range(200):
    A.spmv(x.data_ptr(), y.data_ptr())
e1.record()
torch.cuda.synchronize()
print("us per call", e0.elapsed_time(e1) / 200 * 1e3)
A.free()
