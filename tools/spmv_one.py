"""Run one CSR SpMV kernel on NPB class C a few times (for ncu captures).
    python tools/spmv_one.py [tiled|vector|exact] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402

kern = sys.argv[1] if len(sys.argv) > 1 else "auto"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
N.check(N.lib().b200_init(0))
N.lib().b200_set_kernel(kern.encode())
rp, ci, val = D.gen_npb(150000, 15, 110.0)
A = D.Matrix.csr(rp, ci, val)
x = torch.rand(len(rp) - 1, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    A.spmv(x.data_ptr(), y.data_ptr(), s)
torch.cuda.synchronize()
print("ok", kern, A.info())
