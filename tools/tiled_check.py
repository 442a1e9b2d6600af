"""Correctness of the tiled SpMV variant selected by LILAC_B200_TILED_PROBE
(0 = default, 8 = eight nonzeros per lane) on NPB class C against the oracle
(per-row bound 1e-12 * sum |a x|)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle_lib as O  # noqa: E402
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402

N.check(N.lib().b200_init(0))
N.lib().b200_set_kernel(b"tiled")
rp, ci, val = D.gen_npb(150000, 15, 110.0)
A = D.Matrix.csr(rp, ci, val)
xh = np.random.default_rng(5).uniform(-1, 1, 150000)
x = torch.from_numpy(xh).cuda()
y = torch.empty_like(x)
A.spmv(x.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
ref = O.spmv_csr_mt(rp, ci, val, xh)
scale = O.spmv_csr_mt(rp, ci, np.abs(val), np.abs(xh))
err = np.abs(y.cpu().numpy() - ref)
print("mode", os.environ.get("LILAC_B200_TILED_PROBE", "0"), "kernel", A.info()["kernel"],
      "max err/scale", float((err / scale).max()), "ok", bool((err <= 1e-12 * scale).all()))
