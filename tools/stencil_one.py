"""Run the 27-point stencil SpMV (device-generated, N^3 rows) a few times (for ncu captures / timing).
    python tools/stencil_one.py [N] [reps] [kernel]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 420
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kern = sys.argv[3] if len(sys.argv) > 3 else "auto"
N.check(N.lib().b200_init(0))
N.lib().b200_set_kernel(kern.encode())
A = D.Matrix.stencil27(nx)
info = A.info()
x = torch.rand(nx ** 3, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
A.spmv(x.data_ptr(), y.data_ptr(), s)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    A.spmv(x.data_ptr(), y.data_ptr(), s)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
by = info["nnz"] * (8 + info["col_bytes"]) + 16 * info["rows"] + 8 * (info["rows"] + 1) + 8 * info["cols"]
print(f"N={nx} kernel={info['kernel']} lanes={info['lanes']} {ms*1e3:.1f} us {by/ms/1e6:.1f} GB/s frac {by/ms/1e6/6545.9:.3f}")
