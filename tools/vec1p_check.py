"""Parity of the pipelined one-pass vector kernel (k_csr_vector_1p) forced on
small matrices: run with LILAC_B200_VEC_1P=1 (tests/test_gpu_parity.py runs it
in a subprocess). Checks SpMV vs the oracle (1e-12 sum |a x|) on banded,
random short-row and 27-point stencil matrices, and a CG solve on the stencil
(the fused p.q variant)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import oracle_lib as O  # noqa: E402
from paper_2001_07938_b200.workloads import gen_stencil27  # noqa: E402
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402
from paper_2001_07938_b200 import harness as H  # noqa: E402

assert os.environ.get("LILAC_B200_VEC_1P") == "1"
N.check(N.lib().b200_init(0))
N.lib().b200_set_kernel(b"vector")
rng = np.random.default_rng(11)


def check(rp, ci, val):
    rows = len(rp) - 1
    x = rng.uniform(-2, 2, int(ci.max()) + 1 if len(ci) else 1)
    y = np.full(rows, np.nan)
    H.spmv_csr(rows, y, rp, val, x, ci)
    ref = O.spmv_csr(rp, ci, val, x)
    bound = O.spmv_csr(rp, ci, np.abs(val), np.abs(x))
    assert np.all(np.abs(y - ref) <= 1e-12 * bound), "vector 1p parity"


# banded rows of 0..31 nonzeros (max row + 1 <= 4S with S = 8)
rows = 50000
lens = rng.integers(0, 32, rows)
rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
ci = np.concatenate([np.sort(rng.choice(np.arange(max(0, i - 40), min(rows, i + 40)), size=k, replace=False))
                     for i, k in enumerate(lens)]).astype(np.int64)
check(rp, ci, rng.uniform(-2, 2, len(ci)))
rp, ci, val = gen_stencil27(30)
check(rp, ci, val)
# CG on the stencil: the p.q variant
import torch  # noqa: E402
nx = 30
A = D.Matrix.csr(rp, ci, val)
cg = D.CG(A)
b = torch.from_numpy(rng.uniform(-1, 1, nx ** 3)).cuda()
z = torch.empty_like(b)
res = cg.solve(b.data_ptr(), 40, z.data_ptr())
torch.cuda.synchronize()
zh = z.cpu().numpy()
true_res = np.linalg.norm(b.cpu().numpy() - O.spmv_csr(rp, ci, val, zh))
assert abs(res - true_res) <= 1e-9 * np.linalg.norm(b.cpu().numpy()), (res, true_res)
print("vec1p ok")
