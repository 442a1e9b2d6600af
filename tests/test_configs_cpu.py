"""CPU checks of the benchmark input synthesis (tools/bench_configs.py):
the JDS encoder equals the oracle's jds_from_dense contract bit-for-bit, and
the stencil/Kronecker generators produce the named shapes."""
import os
import sys

import numpy as np

import oracle_lib as O

sys.path.insert(0, os.path.join(O.ROOT, "tools"))
import bench_configs as B  # noqa: E402


def test_parboil_shape_and_jds_encoder_bit_exact():
    rp, ci, val = B.gen_parboil()
    assert len(rp) - 1 == 146_000 and abs(rp[-1] - 1_500_000) < 30_000
    assert np.diff(rp).min() >= 1 and np.diff(rp).max() <= 64
    got = B.csr_to_jds(rp, ci, val)
    want = O.jds_from_csr(rp, ci, val)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_stencil27_shape():
    nx = 6
    rp, ci, val = B.gen_stencil27(nx)
    assert rp[-1] == (3 * nx - 2) ** 3
    assert np.diff(rp).max() == 27
    x = np.ones(nx ** 3)
    y = O.spmv_csr(rp, ci, val, x)
    # interior rows: 26.1 - 26 = 0.1
    assert abs(y[(nx // 2) * nx * nx + (nx // 2) * nx + nx // 2] - 0.1) < 1e-12


def test_kronecker_column_stochastic():
    rp, ci, val = B.gen_kronecker(10)
    n = len(rp) - 1
    assert n == 1024 and rp[-1] == 16 * 1024
    colsum = np.bincount(ci, weights=val, minlength=n)
    nz = np.bincount(ci, minlength=n) > 0
    assert np.allclose(colsum[nz], 1.0)
