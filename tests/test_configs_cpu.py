"""CPU checks of the benchmark input synthesis (paper_2001_07938_b200/workloads.py):
the JDS encoder equals the oracle's jds_from_dense contract bit-for-bit, and
the stencil/Kronecker generators produce the named shapes."""
import os
import sys

import numpy as np

import oracle_lib as O

from paper_2001_07938_b200 import workloads as B  # noqa: E402


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


def test_stencil_rows_match_whole_and_rowsum():
    nx = 7
    rp, ci, val = B.gen_stencil27(nx)
    r0, r1 = 50, 200
    srp, sci, sval = B.gen_stencil27_rows(nx, r0, r1)
    assert np.array_equal(srp, rp[r0:r1 + 1] - rp[r0])
    assert np.array_equal(sci, ci[rp[r0]:rp[r1]]) and np.array_equal(sval, val[rp[r0]:rp[r1]])
    y = O.spmv_csr(rp, ci, val, np.ones(nx ** 3))
    assert np.array_equal(B.stencil27_rowsum(nx, r0, r1), y[r0:r1])
    assert B.stencil27_nnz(nx) == rp[-1]


def test_stencil_prefix_and_shard_bounds():
    """The closed-form prefix count (used for the shard bounds) against the
    generated rows, and the bounds against the oracle's nnz-balanced row
    partition of the same matrix (the sharded driver's partition)."""
    for nx in (1, 2, 3, 6):
        rp, _, _ = B.gen_stencil27(nx)
        assert [B.stencil27_prefix_nnz(nx, r) for r in range(nx ** 3 + 1)] == list(rp)
    nx = 12
    rp, _, _ = B.gen_stencil27(nx)
    for k in (1, 2, 3, 5, 8):
        assert np.array_equal(B.stencil27_bounds(nx, k), O.partition_rows(rp, k)), k


def test_jds_slices_reproduce_whole_bitwise():
    rp, ci, val = B.gen_parboil(n=5000, nnz_target=50_000)
    perm, nzcnt, jd_ptr, jval, jcol = B.csr_to_jds(rp, ci, val)
    x = np.random.default_rng(3).uniform(-1, 1, 5000)
    whole = O.spmv_jds(nzcnt, perm, jval, jd_ptr, x, jcol)
    out = np.full(5000, np.nan)
    for j0, j1 in ((0, 1234), (1234, 1235), (1235, 5000)):
        snz, sperm, sv, sptr, sc, orig = B.jds_slice(nzcnt, perm, jval, jd_ptr, jcol, j0, j1)
        out[orig] = O.spmv_jds(snz, sperm, sv, sptr, x, sc)
    assert O.same_bits(out, whole)
    assert O.same_bits(O.spmv_jds_mt(nzcnt, perm, jval, jd_ptr, x, jcol, 4), whole)


def test_native_npb_outer_matches_benchmark_loop():
    rp, ci, val = O.npb_makea(1400, 7, 10.0)
    ref_zeta, ref_rn = O.npb_cg(rp, ci, val, 15, 10.0)
    it = O.NpbOuter(rp, ci, val, 10.0, nthreads=3)
    it.step()
    it.x[:] = 1.0
    for _ in range(15):
        zeta, rn = it.step()
    assert zeta == ref_zeta and rn == ref_rn


def test_kronecker_native_matches_restatement():
    for scale in (5, 8):
        got = B.gen_kronecker(scale)
        want = B.gen_kronecker_reference(scale)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)
