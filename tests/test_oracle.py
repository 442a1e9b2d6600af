"""Pin the oracle (oracle/oracle.c) against the reference's own outputs.

The golden fixtures in tests/golden/ were written by oracle/make_golden.cpp,
which replays the reference test suites' seeded generators and records what the
reference CPU harness (src/interp.cpp:330-389) returned. Bit-exact throughout.
"""
import numpy as np
import pytest

import oracle_lib as O


@pytest.mark.parametrize("name,case", O.all_golden_cases(), ids=lambda v: v if isinstance(v, str) else "")
def test_oracle_matches_reference_golden(name, case):
    c = O.case_arrays(case)
    # encoders (oracles.hpp:68-144) are bit-exact index work
    rp, ci, val = O.csr_from_dense(c["dense"])
    assert np.array_equal(rp, c["row_ptr"]) and np.array_equal(ci, c["col_ind"])
    assert O.same_bits(val, c["val"])
    perm, nzcnt, jd_ptr, jval, jcol = O.jds_from_csr(rp, ci, val)
    assert np.array_equal(perm, c["perm"])
    assert np.array_equal(nzcnt, c["nzcnt"])
    assert np.array_equal(jd_ptr, c["jd_ptr"])
    assert np.array_equal(jcol, c["jds_col_ind"])
    assert O.same_bits(jval, c["jds_val"])
    # computations (what_interp.cpp:87-108): bit-exact vs the reference harness
    y = O.spmv_csr(c["row_ptr"], c["col_ind"], c["val"], c["x"])
    assert O.same_bits(y, c["y_csr"])
    yj = O.spmv_jds(c["nzcnt"], c["perm"], c["jds_val"], c["jd_ptr"], c["x"], c["jds_col_ind"])
    assert O.same_bits(yj, c["y_jds"])
    # the reference's dense brute force agrees (test_what.cpp:84-95 property)
    assert O.same_bits(y, c["y_dense"])


def test_sample5_frozen_arrays():
    s = O.golden("sample5.json")
    fz = s["frozen"]
    assert s["ones"]["csr"]["val"] == fz["csr_val"]
    assert s["ones"]["jds"]["perm"] == fz["jds_perm"]
    assert s["ones"]["jds"]["jd_ptr"] == fz["jds_jd_ptr"]
    assert s["ones"]["y_csr"] == fz["y_ones"] == [2, 4, 4, 2, 0]
    assert s["counting"]["y_csr"] == fz["y_counting"] == [4, 12, 15, 8, 2]


def test_dot_golden():
    for c in O.golden("dot_seed5150.json")["cases"]:
        a = np.array(c["a"], np.float64)
        b = np.array(c["b"], np.float64)
        r = O.dot(a, b)
        assert O.same_bits(np.array([r]), np.array([c["result"]]))
    # empty range leaves an exact +0.0 (test_what.cpp:126-131)
    r = O.dot(np.zeros(0), np.zeros(0))
    assert r == 0.0 and not np.signbit(r)


def test_fnv1a_vectors():
    for s, h in O.golden("abi.json")["fnv1a"]:
        assert O.fnv1a(s.encode()) == h


def test_out_of_bounds_is_reported():
    rp = np.array([0, 2], np.int64)
    ci = np.array([0, 7], np.int64)
    with pytest.raises(IndexError):
        O.spmv_csr(rp, ci, np.ones(2), np.ones(3))


def test_partition_rows_properties():
    rng = np.random.default_rng(1)
    lens = rng.integers(0, 50, size=1000)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    for k in (1, 2, 3, 4, 8):
        b = O.partition_rows(rp, k)
        assert b[0] == 0 and b[-1] == 1000
        assert np.all(np.diff(b) >= 0)
        nnz = rp[-1]
        for g in range(1, k):
            # first row boundary at or past the g-th nnz quantile
            t = (nnz * g + k - 1) // k
            assert rp[b[g]] >= t
            assert b[g] == 0 or rp[b[g] - 1] < t or b[g] == b[g - 1]


def test_npb_cg_class_s_zeta():
    # NPB 3.x class S: na=1400, nonzer=7, niter=15, shift=10, zeta_verify
    rp, ci, val = O.npb_makea(1400, 7, 10.0)
    assert rp[-1] == 78148
    zeta, _ = O.npb_cg(rp, ci, val, 15, 10.0)
    assert abs(zeta - 8.5971775078648) / 8.5971775078648 <= 1e-10


def test_npb_cg_class_a_zeta():
    rp, ci, val = O.npb_makea(14000, 11, 20.0)
    assert rp[-1] == 1853104
    zeta, _ = O.npb_cg(rp, ci, val, 15, 20.0)
    assert abs(zeta - 17.130235054029) / 17.130235054029 <= 1e-10


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_matches_reference_harness_at_scale():
    """Larger seeded matrices (ragged rows, empty rows, long rows) through the
    reference's own HarnessFn vs the oracle: bit-exact."""
    import ctypes as C
    R = O.ref()
    rng = np.random.default_rng(20240817)
    for rows, maxlen in ((1, 0), (3000, 40), (500, 900)):
        lens = rng.integers(0, maxlen + 1, size=rows)
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        nnz = int(rp[-1])
        cols = max(rows, 1)
        ci = np.sort(rng.integers(0, cols, size=nnz)).astype(np.int64)
        val = rng.uniform(-2, 2, size=nnz)
        x = rng.uniform(-2, 2, size=cols)
        h = R.ref_prepare_csr(rows, O.ptr(rp), O.ptr(val), O.ptr(x), O.ptr(ci), nnz, cols)
        assert R.ref_call(h) == 0
        yr = np.zeros(rows)
        R.ref_output(h, O.ptr(yr))
        R.ref_free(h)
        assert O.same_bits(O.spmv_csr(rp, ci, val, x), yr)
        assert O.same_bits(O.spmv_csr_mt(rp, ci, val, x, 4), yr)
    # the reference rejects out-of-range columns with OutOfBounds
    rp = np.array([0, 1], np.int64)
    ci = np.array([5], np.int64)
    h = R.ref_prepare_csr(1, O.ptr(rp), O.ptr(np.ones(1)), O.ptr(np.ones(2)), O.ptr(ci), 1, 2)
    assert R.ref_call(h) == -1
    assert b"OutOfBounds" in R.ref_last_error()
    R.ref_free(h)
    del C


def test_oracle_gemm_matches_reference_harness_golden():
    """orc_gemm vs the reference's lilac.gemm HarnessFn outputs
    (test_interp.cpp:276-297 trials, seed 424242): bit-exact."""
    cases = O.golden("interp_harness_seed424242.json")["cases"]
    for c in cases:
        g = c["gemm"]
        out = O.gemm(g["n"], g["m"], g["p"], np.array(g["a"], np.float64), np.array(g["b"], np.float64))
        assert O.same_bits(out, np.array(g["c"], np.float64))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_npb_class_a_zeta_through_reference_harness():
    """SURVEY §8(d) input 1: NPB CG class A whose SpMVs and dot products are
    the reference's own lilac.spmv_csr / lilac.dotproduct HarnessFns
    (interp.cpp:330-389, oracle/_ref), host vector updates; zeta verified to
    NPB's 1e-10 (warm-up iteration + 15, ~40 s on 8 threads)."""
    rp, ci, val = O.npb_makea(14000, 11, 20.0)
    cg = O.RefNpbCG(rp, ci, val, 20.0)
    try:
        cg.step()
        cg.x[:] = 1.0
        for _ in range(15):
            zeta, rnorm = cg.step()
    finally:
        cg.free()
    assert abs(zeta - 17.130235054029) / 17.130235054029 <= 1e-10
    assert cg.spmvs == 16 * 26
