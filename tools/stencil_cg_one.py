"""A few CG steps on the 27-point stencil (device-generated) — for ncu launch lists.
    python tools/stencil_cg_one.py [N] [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 420
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N.check(N.lib().b200_init(0))
A = D.Matrix.stencil27(nx)
cg = D.CG(A)
ones = torch.ones(nx ** 3, dtype=torch.float64, device="cuda")
b = torch.empty_like(ones)
A.spmv(ones.data_ptr(), b.data_ptr())
z = torch.empty_like(ones)
r = cg.solve(b.data_ptr(), iters, z.data_ptr())
torch.cuda.synchronize()
print("residual", r)
