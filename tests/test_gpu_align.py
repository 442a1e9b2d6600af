"""Odd-element sub-ranges through the harness and the device API (B200 only).

Vectors handed to the library may be any 8-byte-aligned view: a sub-range of a
device mirror after a write-back (`dot(y+1, y+1, n-1)`), or a torch slice
`x[1:]` passed to the device API. The 16-byte vector loads of the dot and the
bulk copies of the tiled SpMV's x slabs must not fault on them (a misaligned
address is a sticky error that kills the CUDA context), and the results must
match the oracle.
"""
import numpy as np
import pytest

import oracle_lib as O
from paper_2001_07938_b200 import _native as N
from paper_2001_07938_b200 import device as D
from paper_2001_07938_b200 import harness as H

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _mode():
    H.set_errors_return(True)
    N.lib().b200_set_kernel(b"auto")
    yield
    N.lib().b200_set_kernel(b"auto")


def _matrix(n, seed, per_row=24):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, per_row, n)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = rng.integers(0, n, int(rp[-1])).astype(np.int64)
    for i in range(n):
        ci[rp[i]:rp[i + 1]].sort()
    val = rng.uniform(-2, 2, int(rp[-1]))
    return rp, ci, val


@pytest.mark.parametrize("off", [1, 3])
def test_dot_on_mirror_subrange(off):
    """y is written back by the SpMV (a device mirror is published); the dots
    then read y[off:] -> a mirror view at an odd element offset."""
    n = 40000
    rp, ci, val = _matrix(n, 11)
    x = np.random.default_rng(12).uniform(-1, 1, n)
    y = np.zeros(n)
    H.spmv_csr(n, y, rp, val, x, ci)
    a = y[off:]
    b = x[off:]
    d = H.dotproduct(n - off, a, a)
    assert abs(d - O.dot(a, a)) <= 1e-12 * O.dot(np.abs(a), np.abs(a))
    d2 = H.dotproduct(n - off, a, b)  # parities of the two views differ
    assert abs(d2 - O.dot(a, b)) <= 1e-12 * O.dot(np.abs(a), np.abs(b))
    d3 = H.dotproduct(n - off - 1, y[off + 1:], y[off:-1])
    ref = O.dot(y[off + 1:], y[off:-1])
    assert abs(d3 - ref) <= 1e-12 * O.dot(np.abs(y[off + 1:]), np.abs(y[off:-1]))


def test_device_api_odd_slices():
    import torch
    n = 50000
    rp, ci, val = _matrix(n, 21)
    N.lib().b200_set_kernel(b"tiled")
    A = D.Matrix.csr(rp, ci, val)
    try:
        assert A.info()["kernel"] == 4, "tiled layout forced"
        xs = torch.rand(n + 1, dtype=torch.float64, device="cuda")
        x = xs[1:]  # 8 bytes past a 256-byte allocation: not 16-byte aligned
        assert x.data_ptr() % 16 == 8
        ys = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
        y = ys[1:]
        A.spmv(x.data_ptr(), y.data_ptr())
        torch.cuda.synchronize()
        xh = x.cpu().numpy()
        ref = O.spmv_csr(rp, ci, val, xh)
        bound = O.spmv_csr(rp, ci, np.abs(val), np.abs(xh))
        assert np.all(np.abs(y.cpu().numpy() - ref) <= 1e-12 * bound)
        out = torch.zeros(2, dtype=torch.float64, device="cuda")
        D.dot(x.data_ptr(), y.data_ptr(), n, out.data_ptr())
        D.dot(x.data_ptr(), ys[:n].data_ptr(), n, out[1:].data_ptr())
        torch.cuda.synchronize()
        yh = y.cpu().numpy()
        assert abs(out[0].item() - O.dot(xh, yh)) <= 1e-12 * O.dot(np.abs(xh), np.abs(yh))
        y0 = ys[:n].cpu().numpy()
        assert abs(out[1].item() - O.dot(xh, y0)) <= 1e-12 * O.dot(np.abs(xh), np.abs(y0))
        # the context is still healthy after the odd views
        torch.cuda.synchronize()
    finally:
        A.free()
