"""GPU parity of the B200 harness path against the oracle (B200 only).

Every call goes through the C ABI (liblilac_b200.so). Bars:
  * exact CSR kernel, JDS kernel, axpy/xpay, exact dot: bit-identical to the
    reference CPU harness (golden fixtures written by the reference itself) and
    to the oracle restatement pinned to it;
  * fast CSR kernel and fast dot: |y - y_ref| <= TOL * sum_j |a_ij x_j| per
    element, TOL = 1e-12 (north star: "1e-12 for fp64 SpMV"), exact zero when
    the row has no nonzero products;
  * NPB CG: zeta within 1e-10 relative of NPB's official value.
"""
import zlib

import numpy as np
import pytest

import oracle_lib as O
from paper_2001_07938_b200 import _native as N
from paper_2001_07938_b200 import device as D
from paper_2001_07938_b200 import harness as H

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(autouse=True)
def _mode():
    H.set_errors_return(True)
    N.lib().b200_set_kernel(b"auto")
    N.lib().b200_set_exact_blas(0)
    yield
    N.lib().b200_set_kernel(b"auto")
    N.lib().b200_set_exact_blas(0)


def spmv_bound(rp, ci, val, x):
    """sum_j |a_ij x_j| per row (the standard SpMV error-bound scale)."""
    rows = len(rp) - 1
    return O.spmv_csr(rp, ci, np.abs(val), np.abs(x)[: max(1, len(x))], rows) if rows else np.zeros(0)


def assert_within(y, y_ref, scale, tol=TOL):
    err = np.abs(y - y_ref)
    bad = err > tol * scale
    assert not bad.any(), f"{bad.sum()} rows exceed tol; worst {np.max(err / np.maximum(scale, 1e-300))}"


def run_csr(rp, ci, val, x, rows=None):
    rows = len(rp) - 1 if rows is None else rows
    y = np.full(rows, np.nan)
    H.spmv_csr(rows, y, rp, val, x, ci)
    return y


# --------------------------------------------------------------------------------
# golden fixtures (reference outputs)
# --------------------------------------------------------------------------------

@pytest.mark.parametrize("name,case", O.all_golden_cases(), ids=lambda v: v if isinstance(v, str) else "")
def test_golden_csr_exact_bitwise(name, case):
    c = O.case_arrays(case)
    N.lib().b200_set_kernel(b"exact")
    y = run_csr(c["row_ptr"], c["col_ind"], c["val"], c["x"])
    assert O.same_bits(y, c["y_csr"])


@pytest.mark.parametrize("name,case", O.all_golden_cases(), ids=lambda v: v if isinstance(v, str) else "")
def test_golden_csr_fast_within_tolerance(name, case):
    c = O.case_arrays(case)
    y = run_csr(c["row_ptr"], c["col_ind"], c["val"], c["x"])
    assert_within(y, c["y_csr"], spmv_bound(c["row_ptr"], c["col_ind"], c["val"], c["x"]))


@pytest.mark.parametrize("name,case", O.all_golden_cases(), ids=lambda v: v if isinstance(v, str) else "")
def test_golden_csr_tiled_within_tolerance(name, case):
    c = O.case_arrays(case)
    N.lib().b200_set_kernel(b"tiled")
    y = run_csr(c["row_ptr"], c["col_ind"], c["val"], c["x"])
    assert_within(y, c["y_csr"], spmv_bound(c["row_ptr"], c["col_ind"], c["val"], c["x"]))


@pytest.mark.parametrize("name,case", O.all_golden_cases(), ids=lambda v: v if isinstance(v, str) else "")
def test_golden_csr_merge_within_tolerance(name, case):
    c = O.case_arrays(case)
    N.lib().b200_set_kernel(b"merge")
    y = run_csr(c["row_ptr"], c["col_ind"], c["val"], c["x"])
    assert_within(y, c["y_csr"], spmv_bound(c["row_ptr"], c["col_ind"], c["val"], c["x"]))


@pytest.mark.parametrize("name,case", O.all_golden_cases(), ids=lambda v: v if isinstance(v, str) else "")
def test_golden_csr_split_within_tolerance(name, case):
    c = O.case_arrays(case)
    N.lib().b200_set_kernel(b"split")
    y = run_csr(c["row_ptr"], c["col_ind"], c["val"], c["x"])
    assert_within(y, c["y_csr"], spmv_bound(c["row_ptr"], c["col_ind"], c["val"], c["x"]))


@pytest.mark.parametrize("name,case", O.all_golden_cases(), ids=lambda v: v if isinstance(v, str) else "")
def test_golden_csr_lane_within_tolerance(name, case):
    c = O.case_arrays(case)
    N.lib().b200_set_kernel(b"lane")
    y = run_csr(c["row_ptr"], c["col_ind"], c["val"], c["x"])
    assert_within(y, c["y_csr"], spmv_bound(c["row_ptr"], c["col_ind"], c["val"], c["x"]))


@pytest.mark.parametrize("name,case", O.all_golden_cases(), ids=lambda v: v if isinstance(v, str) else "")
def test_golden_jds_bitwise(name, case):
    c = O.case_arrays(case)
    y = np.full(c["rows"], np.nan)
    H.spmv_jds(c["rows"], y, c["nzcnt"], c["perm"], c["jds_val"], c["jd_ptr"], c["x"], c["jds_col_ind"])
    assert O.same_bits(y, c["y_jds"])


def test_golden_sample5():
    s = O.golden("sample5.json")
    for key, want in (("ones", [2, 4, 4, 2, 0]), ("counting", [4, 12, 15, 8, 2])):
        c = O.case_arrays(s[key])
        y = run_csr(c["row_ptr"], c["col_ind"], c["val"], c["x"])
        assert y.tolist() == want


def test_golden_dot():
    cases = O.golden("dot_seed5150.json")["cases"]
    for exact in (1, 0):
        N.lib().b200_set_exact_blas(exact)
        for c in cases:
            a = np.array(c["a"], np.float64)
            b = np.array(c["b"], np.float64)
            r = H.dotproduct(len(a), a, b)
            if exact:
                assert O.same_bits(np.array([r]), np.array([c["result"]]))
            else:
                assert abs(r - c["result"]) <= TOL * float(np.sum(np.abs(a * b))) or r == c["result"]
    r = H.dotproduct(0, np.zeros(0), np.zeros(0))
    assert r == 0.0 and not np.signbit(r)


# --------------------------------------------------------------------------------
# seeded random matrices at scale (vs the pinned oracle)
# --------------------------------------------------------------------------------

def random_csr(rng, rows, cols, lens):
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(rp[-1])
    ci = np.empty(nnz, np.int64)
    for i in range(rows):
        k = lens[i]
        if k:
            ci[rp[i]:rp[i + 1]] = np.sort(rng.choice(cols, size=min(k, cols), replace=k > cols))
    val = rng.uniform(-2, 2, nnz)
    return rp, ci, val


SHAPES = {
    "short_rows": (20000, 20000, lambda r, n: r.integers(0, 8, n)),
    "npb_like": (3000, 3000, lambda r, n: r.integers(150, 330, n)),
    "stencil_like": (30000, 30000, lambda r, n: np.full(n, 27)),
    "skewed": (5000, 5000, lambda r, n: np.minimum(r.zipf(1.6, n), 4000)),
    "long_rows": (40, 200000, lambda r, n: r.integers(5000, 60000, n)),
    "empty_rows": (1000, 1000, lambda r, n: np.where(r.random(n) < 0.5, 0, r.integers(1, 40, n))),
}


@pytest.mark.parametrize("shape", sorted(SHAPES))
def test_random_csr_vs_oracle(shape):
    rows, cols, lens_fn = SHAPES[shape]
    rng = np.random.default_rng(zlib.crc32(shape.encode()))
    lens = np.asarray(lens_fn(rng, rows), np.int64)
    rp, ci, val = random_csr(rng, rows, cols, lens)
    x = rng.uniform(-2, 2, cols)
    y_ref = O.spmv_csr(rp, ci, val, x)
    y = run_csr(rp, ci, val, x)
    assert_within(y, y_ref, spmv_bound(rp, ci, val, x))
    for kernel in (b"vector", b"tiled", b"merge", b"split", b"lane"):
        N.lib().b200_set_kernel(kernel)
        assert_within(run_csr(rp, ci, val, x), y_ref, spmv_bound(rp, ci, val, x))
    N.lib().b200_set_kernel(b"exact")
    assert O.same_bits(run_csr(rp, ci, val, x), y_ref)
    # JDS of the same matrix (encoder pinned to oracles.hpp:109-144): bit-exact
    perm, nzcnt, jd_ptr, jval, jcol = O.jds_from_csr(rp, ci, val)
    yj = np.full(rows, np.nan)
    H.spmv_jds(rows, yj, nzcnt, perm, jval, jd_ptr, x, jcol)
    assert O.same_bits(yj, y_ref)


def _short_rows_csr(rng, rows, cols, max_len):
    """Vectorised random CSR: row lengths in [0, max_len], distinct sorted columns."""
    lens = rng.integers(0, max_len + 1, rows).astype(np.int64)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(rp[-1])
    row = np.repeat(np.arange(rows, dtype=np.int64), lens)
    ci = rng.integers(0, cols, nnz).astype(np.int64)
    order = np.lexsort((ci, row))
    ci = ci[order]
    dup = np.zeros(nnz, bool)
    dup[1:] = (row[1:] == row[:-1]) & (ci[1:] == ci[:-1])
    ci[dup] = (ci[dup] + 1) % cols  # rare; keep rows sorted enough for the reference semantics
    return rp, ci, rng.uniform(-2, 2, nnz)


def test_tiled_layout_edge_cases():
    """Tiled layout (tcsr_build.cpp) corners: more tiles than SMs (several per
    CTA), rows of 0-3 nonzeros (empty rows inside runs -> zero entries, several
    row starts per 4-nonzero chunk, lanes without chunks in short runs), an odd
    column count (odd last slab), and an Inf in x: rows that do not reference
    it must stay finite (padding entries read the zero cell, never x)."""
    rng = np.random.default_rng(20240817)
    rows, cols = 148 * 4096 + 5000, 2 * 12288 + 1
    rp, ci, val = _short_rows_csr(rng, rows, cols, 3)
    x = rng.uniform(-2, 2, cols)
    x[cols - 1] = np.inf
    y_ref = O.spmv_csr(rp, ci, val, x)
    N.lib().b200_set_kernel(b"tiled")
    A = D.Matrix.csr(rp, ci, val)
    assert A.info()["kernel"] == 4 and A.info()["col_bytes"] == 2
    A.free()
    y = run_csr(rp, ci, val, x)
    fin = np.isfinite(y_ref)
    assert (~fin).sum() > 0 and fin.sum() > rows // 2
    assert np.array_equal(np.isfinite(y), fin)
    assert np.array_equal(y[~fin], y_ref[~fin])  # same signed infinities
    assert_within(y[fin], y_ref[fin], spmv_bound(rp, ci, val, np.where(np.isfinite(x), x, 0.0))[fin])


def test_fused_cg_is_deterministic_run_to_run():
    """The fused CG kernel's dots use a fixed per-CTA partition summed in CTA
    order, and the tiled SpMV's row sums a fixed layout order: two runs give
    the same bits."""
    na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES["A"]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    N.lib().b200_set_kernel(b"tiled")
    A = D.Matrix.csr(rp, ci, val)
    assert A.info()["kernel"] == 4
    got = []
    for _ in range(2):
        cg = D.CG(A)
        got.append(cg.npb(niter, shift))
        cg.free()
    A.free()
    assert got[0] == got[1], got
    assert abs(got[0][0] - zeta_ref) / zeta_ref <= 1e-10


@pytest.mark.parametrize("parts", [1, 2, 3, 4])
def test_tiled_slab_parts(parts, monkeypatch):
    """Tiles cut into slab parts (TcsrDev::parts: one CTA per part, the last
    part of a tile adds the parts in order): SpMV within tolerance of the
    oracle, and NPB class A CG (the fused kernel's DOT path and the per-step
    kernels) verifies zeta, for every part count."""
    monkeypatch.setenv("LILAC_B200_TILE_PARTS", str(parts))
    na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES["A"]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    N.lib().b200_set_kernel(b"tiled")
    x = np.random.default_rng(parts).uniform(-1, 1, na)
    y = run_csr(rp, ci, val, x)
    assert_within(y, O.spmv_csr(rp, ci, val, x), spmv_bound(rp, ci, val, x))
    y2 = run_csr(rp, ci, val, x)  # the tickets were reset by the last part
    assert np.array_equal(y, y2)
    A = D.Matrix.csr(rp, ci, val)
    assert A.info()["kernel"] == 4
    cg = D.CG(A)  # one GPU: the fused persistent kernel
    zeta, _ = cg.npb(niter, shift)
    cg.free()
    A.free()
    assert abs(zeta - zeta_ref) / zeta_ref <= 1e-10, (parts, zeta)
    d = D.DistCG.local(2, rp, ci, val)  # shards: the per-step tiled kernel with the p.q partials
    assert all(d.info(g)["tiled"] for g in range(2))
    zeta2, _ = d.npb(niter, shift)
    d.free()
    assert abs(zeta2 - zeta_ref) / zeta_ref <= 1e-10, (parts, zeta2)
    # a ragged matrix: empty rows, rows spanning slabs, fewer slabs than parts
    rng = np.random.default_rng(40 + parts)
    for cols in (3000, 100_000):
        rp2, ci2, val2 = random_csr(rng, 20000, cols, rng.integers(0, 120, 20000) * (rng.random(20000) < 0.8))
        x2 = rng.uniform(-1, 1, cols)
        y2 = run_csr(rp2, ci2, val2, x2)
        assert_within(y2, O.spmv_csr(rp2, ci2, val2, x2), spmv_bound(rp2, ci2, val2, x2))


def test_fused_cg_matches_per_step_kernels():
    """CG on one GPU with the tiled layout runs its steps in one persistent
    cooperative kernel (k_cg_tiled) — here with more tiles than SMs; the vector
    layout runs three kernels per step. Same iterates up to rounding."""
    import torch
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from paper_2001_07938_b200.workloads import gen_stencil27
    nx = 85  # 614,125 rows > 148 x 4096
    rp, ci, val = gen_stencil27(nx)
    n = nx ** 3
    b = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, n)).cuda()
    out = {}
    for kern in (b"tiled", b"vector"):
        N.lib().b200_set_kernel(kern)
        A = D.Matrix.csr(rp, ci, val)
        assert (A.info()["kernel"] == 4) == (kern == b"tiled")
        cg = D.CG(A)
        z = torch.empty_like(b)
        res = cg.solve(b.data_ptr(), 30, z.data_ptr())
        torch.cuda.synchronize()
        out[kern] = (res, z.cpu().numpy())
        cg.free()
        A.free()
    (r_t, z_t), (r_v, z_v) = out[b"tiled"], out[b"vector"]
    bn = float(torch.linalg.norm(b))
    assert r_v < 0.01 * bn  # CG made progress (kappa ~ 500: not converged in 30 steps)
    assert abs(r_t - r_v) <= 1e-8 * r_v
    assert np.abs(z_t - z_v).max() <= 1e-9 * np.abs(z_v).max()


def test_vector_one_pass_kernel_forced():
    """The pipelined one-pass vector kernel is chosen only for matrices over
    8 GB; tools/vec1p_check.py forces it (LILAC_B200_VEC_1P=1, read once per
    process, hence the subprocess) on small banded/stencil matrices."""
    import subprocess
    import sys
    import os
    env = dict(os.environ, LILAC_B200_VEC_1P="1")
    r = subprocess.run([sys.executable, os.path.join(O.ROOT, "tools", "vec1p_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "vec1p ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_edge_cases():
    # rows = 0
    y = np.zeros(0)
    H.spmv_csr(0, y, np.zeros(1, np.int64), np.zeros(0), np.zeros(0), np.zeros(0, np.int64))
    # all rows empty
    y = run_csr(np.zeros(11, np.int64), np.zeros(0, np.int64), np.zeros(0), np.zeros(0))
    assert np.all(y == 0) and not np.signbit(y).any()
    # row_ptr not starting at 0: leading nonzeros are simply not addressed
    rp = np.array([3, 5, 6], np.int64)
    ci = np.array([9, 9, 9, 0, 1, 1], np.int64)
    val = np.array([7.0, 7, 7, 1, 2, 4])
    x = np.array([10.0, 100] + [0] * 8)
    assert run_csr(rp, ci, val, x).tolist() == [210.0, 400.0]
    # non-monotone row_ptr: the reference treats the row as empty
    rp = np.array([0, 2, 1, 3], np.int64)
    ci = np.array([0, 1, 2], np.int64)
    val = np.array([1.0, 2, 3])
    x = np.array([1.0, 1, 1])
    assert run_csr(rp, ci, val, x).tolist() == O.spmv_csr(rp, ci, val, x).tolist() == [3.0, 0.0, 5.0]
    # one very long row
    n = 300000
    rng = np.random.default_rng(0)
    rp = np.array([0, n], np.int64)
    ci = np.arange(n, dtype=np.int64)
    val = rng.uniform(-1, 1, n)
    x = rng.uniform(-1, 1, n)
    assert_within(run_csr(rp, ci, val, x), O.spmv_csr(rp, ci, val, x), spmv_bound(rp, ci, val, x))


def test_out_of_bounds_is_an_error_not_a_fallback():
    rp = np.array([0, 2], np.int64)
    ci = np.array([0, -1], np.int64)
    y = np.full(1, 123.0)
    with pytest.raises(H.B200Error) as e:
        H.spmv_csr(1, y, rp, np.ones(2), np.ones(2), ci)
    assert e.value.code == "OutOfBounds"
    assert y[0] == 123.0
    # JDS: perm outside [0, rows)
    with pytest.raises(H.B200Error) as e:
        H.spmv_jds(2, np.zeros(2), np.array([1, 1], np.int64), np.array([0, 5], np.int64), np.ones(2),
                   np.array([0, 2], np.int64), np.ones(2), np.array([0, 1], np.int64))
    assert e.value.code == "OutOfBounds"


def test_blas1_bitwise():
    rng = np.random.default_rng(7)
    for n in (0, 1, 17, 100003):
        x = rng.uniform(-2, 2, n)
        y = rng.uniform(-2, 2, n)
        want = O.axpy(y, 0.37, x)
        yy = y.copy()
        H.axpy(n, yy, 0.37, x)
        assert O.same_bits(yy, want)
        want = x + (-1.25 * y)  # x + beta*y, separate rounding as in NPB's p = r + beta*p
        yy = y.copy()
        H.xpay(n, yy, -1.25, x)
        assert O.same_bits(yy, want)
        r = H.dotproduct(n, x, y)
        assert abs(r - O.dot(x, y)) <= TOL * float(np.sum(np.abs(x * y))) + 0.0
        N.lib().b200_set_exact_blas(1)
        assert O.same_bits(np.array([H.dotproduct(n, x, y)]), np.array([O.dot(x, y)]))
        N.lib().b200_set_exact_blas(0)


# --------------------------------------------------------------------------------
# marshaling contract through the harness (resident matrix, vector-only traffic)
# --------------------------------------------------------------------------------

def test_resident_matrix_moves_only_vectors():
    rng = np.random.default_rng(11)
    rows = 4096
    rp, ci, val = random_csr(rng, rows, rows, rng.integers(10, 40, rows))
    stats0 = H.region_stats()
    base = {k: v["n_update"] for k, v in stats0.items()}
    h2d0 = {k: v["bytes_h2d"] for k, v in stats0.items()}
    x = np.zeros(rows)
    for call in range(10):
        x[:] = rng.uniform(-1, 1, rows)  # the host rewrites x in place every call
        y = run_csr(rp, ci, val, x)
        assert_within(y, O.spmv_csr(rp, ci, val, x), spmv_bound(rp, ci, val, x))
    st = H.region_stats()
    upd = {k: st[k]["n_update"] - base.get(k, 0) for k in st}
    assert upd["b200_spmv_csr.val"] == 1
    assert upd["b200_spmv_csr.row_ptr"] == 1
    assert upd["b200_spmv_csr.col_ind"] == 1
    assert upd["b200_spmv_csr.x"] == 10
    assert st["b200_spmv_csr.val"]["bytes_h2d"] - h2d0.get("b200_spmv_csr.val", 0) == 8 * len(val)
    assert st["b200_spmv_csr.x"]["streaming"]  # rewritten every call: no longer guarded
    assert not st["b200_spmv_csr.val"]["streaming"]
    # in-place mutation of the resident matrix is seen (never stale)
    x[:] = rng.uniform(-1, 1, rows)
    val[len(val) // 2] += 1.0
    y = run_csr(rp, ci, val, x)
    assert_within(y, O.spmv_csr(rp, ci, val, x), spmv_bound(rp, ci, val, x))
    assert H.region_stats()["b200_spmv_csr.val"]["n_update"] - base.get("b200_spmv_csr.val", 0) == 2
    # edge bytes of a misaligned numpy buffer are hashed (Hybrid): mutate the first element
    val[0] += 1.0
    y = run_csr(rp, ci, val, x)
    assert_within(y, O.spmv_csr(rp, ci, val, x), spmv_bound(rp, ci, val, x))
    # identity change -> destruct + construct
    val2 = val.copy()
    d0 = H.region_stats()["b200_spmv_csr.val"]["n_destruct"]
    run_csr(rp, ci, val2, x)
    assert H.region_stats()["b200_spmv_csr.val"]["n_destruct"] == d0 + 1


# --------------------------------------------------------------------------------
# NPB CG
# --------------------------------------------------------------------------------

@pytest.mark.parametrize("cls,kernel", [("S", b"auto"), ("A", b"auto"), ("A", b"tiled"), ("A", b"vector"),
                                        ("A", b"merge"), ("A", b"split"), ("A", b"lane"), ("C", b"auto"),
                                        ("C", b"vector")])
def test_npb_cg_zeta_device_driver(cls, kernel):
    na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES[cls]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    N.lib().b200_set_kernel(kernel)
    A = D.Matrix.csr(rp, ci, val)
    if cls == "C" and kernel == b"auto":
        assert A.info()["kernel"] == 4  # the tiled layout is chosen for NPB's random columns
    cg = D.CG(A)
    zeta, rnorm = cg.npb(niter, shift)
    assert abs(zeta - zeta_ref) / zeta_ref <= 1e-10, (zeta, zeta_ref)
    assert rnorm < 1e-10
    cg.free()
    A.free()


def test_npb_cg_class_s_through_the_c_abi_harnesses():
    """The LiLAC model: the host program keeps its CG loop; SpMV/dot/axpy are
    replaced by harness calls on host arrays (vectors move every call)."""
    na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES["S"]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    n = na
    x = np.ones(n)
    zeta = 0.0
    h2d0 = H.region_stats().get("b200_spmv_csr.val", {}).get("bytes_h2d", 0)
    for it in range(niter + 1):
        z = np.zeros(n)
        r = x.copy()
        p = r.copy()
        q = np.zeros(n)
        rho = H.dotproduct(n, r, r)
        for _ in range(25):
            H.spmv_csr(n, q, rp, val, p, ci)
            d = H.dotproduct(n, p, q)
            alpha = rho / d
            rho0 = rho
            H.axpy(n, z, alpha, p)
            H.axpy(n, r, -alpha, q)
            rho = H.dotproduct(n, r, r)
            H.xpay(n, p, rho / rho0, r)
        t1 = H.dotproduct(n, x, z)
        t2 = 1.0 / np.sqrt(H.dotproduct(n, z, z))
        if it > 0:
            zeta = shift + 1.0 / t1
        x = t2 * z if it > 0 else np.ones(n)
    assert abs(zeta - zeta_ref) / zeta_ref <= 1e-10
    st = H.region_stats()
    # the matrix moved once; every later call moved only vectors
    assert st["b200_spmv_csr.val"]["bytes_h2d"] - h2d0 == 8 * len(val)


def test_device_api_spmv_and_dot():
    import torch
    rng = np.random.default_rng(5)
    rows = 10000
    rp, ci, val = random_csr(rng, rows, rows, rng.integers(0, 64, rows))
    A = D.Matrix.csr(rp, ci, val)
    info = A.info()
    assert info["rows"] == rows and info["nnz"] == len(val) and info["col_bytes"] == 4
    x = rng.uniform(-1, 1, rows)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty(rows, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    A.spmv(xd.data_ptr(), yd.data_ptr(), s.cuda_stream)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    D.dot(xd.data_ptr(), yd.data_ptr(), rows, out.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    y_ref = O.spmv_csr(rp, ci, val, x)
    assert_within(yd.cpu().numpy(), y_ref, spmv_bound(rp, ci, val, x))
    assert abs(out.item() - O.dot(x, y_ref)) <= 1e-10 * float(np.sum(np.abs(x * y_ref)))
    A.free()


# --------------------------------------------------------------------------------
# row-sharded driver (the multi-GPU algorithm, exercised on one GPU)
# --------------------------------------------------------------------------------

@pytest.mark.parametrize("cls,k", [("S", 1), ("S", 2), ("S", 3), ("A", 2), ("A", 4), ("A", 8), ("C", 8)])
def test_sharded_cg_local_shards(cls, k):
    """k shards on one GPU exchanging by device copies: the same code path as
    the NCCL driver minus the transport. zeta must verify and agree with the
    1-GPU solver to ~1e-12 (only the dot-product association differs)."""
    na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES[cls]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    d = D.DistCG.local(k, rp, ci, val)
    bounds = D.partition_rows(rp, k)
    for g in range(k):
        info = d.info(g)
        assert info["row0"] == bounds[g] and info["rows"] == bounds[g + 1] - bounds[g]
        assert info["nnz"] == rp[bounds[g + 1]] - rp[bounds[g]]
    zeta, rnorm = d.npb(niter, shift)
    assert abs(zeta - zeta_ref) / zeta_ref <= 1e-10, (zeta, zeta_ref)
    A = D.Matrix.csr(rp, ci, val)
    cg = D.CG(A)
    z1, _ = cg.npb(niter, shift)
    assert abs(zeta - z1) <= 1e-12 * abs(z1)
    d.free()
    cg.free()
    A.free()


def test_sharded_cg_nccl_single_rank():
    """NCCL transport with world = 1 (the only topology one GPU allows)."""
    na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES["S"]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    nid = D.DistCG.nccl_id()
    bounds = np.array([0, na], np.int64)
    d = D.DistCG.nccl(0, 1, nid, na, bounds, rp, ci, val)
    zeta, _ = d.npb(niter, shift)
    assert abs(zeta - zeta_ref) / zeta_ref <= 1e-10
    d.free()


@pytest.mark.parametrize("cls,k", [("S", 2), ("A", 3), ("A", 8), ("C", 4)])
def test_sharded_cg_peer_memory_exchange_local(cls, k):
    """Peer-memory exchange between local shards (the kernels the IPC path
    runs between processes): zeta bit-identical to the device-copy exchange
    (same partials, same rank-order sums)."""
    na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES[cls]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    d0 = D.DistCG.local(k, rp, ci, val)
    z0, r0 = d0.npb(niter, shift)
    d0.free()
    d = D.DistCG.local(k, rp, ci, val)
    d.use_p2p_local()
    d.set_fused(False)  # the per-step kernels: same partials as the device-copy exchange
    assert d.transport == "p2p"
    z1, r1 = d.npb(niter, shift)
    assert abs(z1 - zeta_ref) / zeta_ref <= 1e-10
    assert z1 == z0 and r1 == r0
    assert not d.fused
    d.free()


@pytest.mark.parametrize("cls,k", [("A", 1), ("A", 2), ("A", 3), ("A", 8), ("C", 1), ("C", 2), ("C", 4), ("C", 8)])
def test_sharded_cg_fused_persistent_kernel(cls, k):
    """The sharded CG in one persistent kernel (k_cg_tiled_dist): k local
    shards as k CTA groups of one cooperative grid, exchanging p slices and
    the dot partials through each other's peer buffers and epoch flags, as
    the ranks of a multi-GPU run would over NVLink. zeta must verify and
    agree with the 1-GPU solver to ~1e-12 (the dot partitions differ)."""
    na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES[cls]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    N.lib().b200_set_kernel(b"tiled")  # class A shards are small enough for the vector kernel by default
    d = D.DistCG.local(k, rp, ci, val)
    for g in range(k):
        assert d.info(g)["tiled"] == 1
    d.use_p2p_local()
    zeta, rnorm = d.npb(niter, shift)
    assert d.fused
    assert abs(zeta - zeta_ref) / zeta_ref <= 1e-10, (zeta, zeta_ref)
    d.set_fused(False)
    z_steps, _ = d.npb(niter, shift)
    assert not d.fused
    assert abs(zeta - z_steps) <= 1e-12 * abs(z_steps)
    d.free()


def test_sharded_cg_peer_memory_halo_on_a_stencil():
    """Banded rows: each shard pushes only the halo its peers read; the
    sharded CG recurrence still matches the device-copy exchange bit for bit."""
    rp, ci, val = _stencil27_host(16)
    n = len(rp) - 1
    d0 = D.DistCG.local(4, rp, ci, val)
    z0, r0 = d0.npb(3, 0.0)
    d0.free()
    d = D.DistCG.local(4, rp, ci, val)
    d.use_p2p_local()
    z1, r1 = d.npb(3, 0.0)
    assert z1 == z0 and r1 == r0 and np.isfinite(z1)
    d.free()
    assert n == 4096


def test_sharded_cg_peer_memory_ipc_single_rank():
    """The IPC export/attach path with world = 1 (no peer to map; exercises
    cudaIpcGetMemHandle and the switch of transport)."""
    na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES["S"]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    d = D.DistCG.nccl(0, 1, D.DistCG.nccl_id(), na, np.array([0, na], np.int64), rp, ci, val)
    h = d.p2p_export()
    assert len(h) == 208
    d.p2p_attach(h)
    assert d.transport == "p2p"
    zeta, _ = d.npb(niter, shift)
    assert abs(zeta - zeta_ref) / zeta_ref <= 1e-10
    d.free()


def test_sharded_cg_load_x_from_host_matches_reset():
    """b200_dist_cg_load_x (the e2e feed at N > 1): x = 1 from host memory
    gives the outer iteration reset() gives, bit for bit."""
    import torch
    na, nonzer, niter, shift, _ = D.NPB_CLASSES["A"]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    d = D.DistCG.local(3, rp, ci, val)
    d.reset()
    d.outer(shift)
    z_reset, r_reset = d.result()
    x = torch.ones(na, dtype=torch.float64, pin_memory=True)
    d.load_x(x.data_ptr())
    d.outer(shift)
    z_load, r_load = d.result()
    assert z_load == z_reset and r_load == r_reset
    d.free()


def test_device_mirrors_serve_written_back_vectors_and_never_go_stale():
    """A harness output written back to the host is mirrored on the device;
    the next harness that reads those bytes gets them device-to-device, and
    any host write (interior page or hashed edge) invalidates the mirror."""
    rng = np.random.default_rng(31)
    n = 20000
    rp, ci, val = random_csr(rng, n, n, rng.integers(5, 30, n))
    x = rng.uniform(-1, 1, n)
    y = np.zeros(n)
    H.spmv_csr(n, y, rp, val, x, ci)
    st0 = H.harness_stats()["b200_dot"] if "b200_dot" in H.harness_stats() else {"bytes_d2d": 0, "bytes_h2d": 0}
    r1 = H.dotproduct(n, y, y)
    st1 = H.harness_stats()["b200_dot"]
    assert st1["bytes_d2d"] - st0["bytes_d2d"] == 8 * n  # served from the device mirror
    assert st1["bytes_h2d"] - st0["bytes_h2d"] == 0
    assert abs(r1 - O.dot(y, y)) <= 1e-12 * O.dot(y, y)
    for idx in (n // 2, 0, n - 1):  # interior page, head edge, tail edge
        H.spmv_csr(n, y, rp, val, x, ci)  # republish
        y[idx] += 3.0
        r = H.dotproduct(n, y, y)
        assert abs(r - O.dot(y, y)) <= 1e-12 * O.dot(y, y), idx


def test_power_law_rows_choose_split_and_match():
    """Kronecker-like skew (one row of 200k nonzeros among short rows): the
    auto policy builds the split plan (long rows in warp chunks); the forced
    merge-path kernel agrees; results within tolerance and deterministic
    (bit-identical across calls)."""
    rng = np.random.default_rng(99)
    n = 300000
    lens = np.minimum(rng.zipf(2.0, n), 200000).astype(np.int64)
    lens[n // 3] = 200000
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = rng.integers(0, n, int(rp[-1])).astype(np.int64)
    val = rng.uniform(-1, 1, int(rp[-1]))
    x = rng.uniform(-1, 1, n)
    A = D.Matrix.csr(rp, ci, val)
    assert A.info()["kernel"] == 6  # lane-range layout for skewed rows
    A.free()
    y_ref = O.spmv_csr(rp, ci, val, x)
    bound = spmv_bound(rp, ci, val, x)
    for kernel in (b"auto", b"merge", b"split", b"lane"):
        N.lib().b200_set_kernel(kernel)
        y1 = run_csr(rp, ci, val, x)
        y2 = run_csr(rp, ci, val, x)
        assert O.same_bits(y1, y2)
        assert_within(y1, y_ref, bound)


# --------------------------------------------------------------------------------
# workload pieces of the BASELINE configs (SURVEY §8(d) inputs 4 and 5)
# --------------------------------------------------------------------------------

def _stencil27_host(nx):
    """Host restatement of the 27-point operator (tools/bench_configs.py)."""
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from paper_2001_07938_b200.workloads import gen_stencil27
    return gen_stencil27(nx)


@pytest.mark.parametrize("nx", [1, 2, 3, 17])
def test_device_stencil_matches_host_generator(nx):
    import torch
    rp, ci, val = _stencil27_host(nx)
    A = D.Matrix.stencil27(nx)
    info = A.info()
    assert info["rows"] == nx ** 3 and info["nnz"] == len(val) and info["max_row"] == min(27, nx ** 3)
    rng = np.random.default_rng(nx)
    xh = rng.uniform(-1, 1, nx ** 3)
    x = torch.from_numpy(xh).cuda()
    y = torch.empty_like(x)
    N.lib().b200_set_kernel(b"exact")  # read at launch by the device API
    A.spmv(x.data_ptr(), y.data_ptr())
    torch.cuda.synchronize()
    y_ref = O.spmv_csr(rp, ci, val, xh)
    assert_within(y.cpu().numpy(), y_ref, spmv_bound(rp, ci, val, xh))
    A.free()


def test_pagerank_device_matches_host_iteration():
    import torch
    rng = np.random.default_rng(3)
    n = 5000
    src = rng.integers(0, n, 60000)
    dst = rng.integers(0, n, 60000)
    outdeg = np.bincount(src, minlength=n).astype(np.float64)
    order = np.lexsort((src, dst))
    src, dst = src[order], dst[order]
    rp = np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))]).astype(np.int64)
    ci = src.astype(np.int64)
    val = 1.0 / outdeg[src]
    A = D.Matrix.csr(rp, ci, val)
    x = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    w = torch.empty_like(x)
    A.pagerank(0.85, 20, x.data_ptr(), w.data_ptr())
    torch.cuda.synchronize()
    xr = np.full(n, 1.0 / n)
    for _ in range(20):
        xr = 0.85 * O.spmv_csr(rp, ci, val, xr) + 0.15 / n
    assert np.allclose(x.cpu().numpy(), xr, rtol=1e-12, atol=1e-15)
    A.free()


@pytest.mark.parametrize("steps", [20, 21])
def test_pagerank_lane_range_fused_update(steps):
    """The lane-range layout folds the PageRank update into its row stores
    (rows stored in the main kernel, rows crossing units in the fix-up, empty
    rows = the teleport term); an odd step count ends with a copy back into x."""
    import torch
    rng = np.random.default_rng(9)
    n = 20000
    src = rng.integers(0, n, 300000)
    dst = (rng.pareto(1.2, 300000) * 40).astype(np.int64) % n  # skewed in-degrees, many empty rows
    outdeg = np.bincount(src, minlength=n).astype(np.float64)
    order = np.lexsort((src, dst))
    src, dst = src[order], dst[order]
    rp = np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))]).astype(np.int64)
    ci = src.astype(np.int64)
    val = 1.0 / outdeg[src]
    N.lib().b200_set_kernel(b"lane")
    A = D.Matrix.csr(rp, ci, val)
    assert A.info()["kernel"] == 6
    x = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    w = torch.empty_like(x)
    A.pagerank(0.85, steps, x.data_ptr(), w.data_ptr())
    torch.cuda.synchronize()
    xr = np.full(n, 1.0 / n)
    for _ in range(steps):
        xr = 0.85 * O.spmv_csr(rp, ci, val, xr) + 0.15 / n
    xd = x.cpu().numpy()
    assert np.all(np.abs(xd - xr) <= 1e-12 * np.abs(xr) + 1e-18), np.max(np.abs(xd - xr) / np.abs(xr))
    A.free()


def test_cg_solve_on_the_stencil_converges():
    import torch
    nx = 24
    rp, ci, val = _stencil27_host(nx)
    A = D.Matrix.stencil27(nx)
    cg = D.CG(A)
    ones = torch.ones(nx ** 3, dtype=torch.float64, device="cuda")
    b = torch.empty_like(ones)
    A.spmv(ones.data_ptr(), b.data_ptr())
    z = torch.empty_like(ones)
    r50 = cg.solve(b.data_ptr(), 50, z.data_ptr())
    bh = b.cpu().numpy()
    zh = z.cpu().numpy()
    # the reported residual is |b - A z| of the returned z, and CG converged to 1
    assert abs(r50 - np.linalg.norm(bh - O.spmv_csr(rp, ci, val, zh))) <= 1e-9 * np.linalg.norm(bh)
    assert r50 < 1e-8 * np.linalg.norm(bh)
    assert np.abs(zh - 1.0).max() < 1e-8
    cg.free()
    A.free()


# --------------------------------------------------------------------------------
# gemm (kernels.lilac:14-19)
# --------------------------------------------------------------------------------

def test_gemm_exact_bitwise_vs_reference_golden():
    """b200_gemm with exact BLAS vs the reference's lilac.gemm outputs."""
    N.lib().b200_set_exact_blas(1)
    for c in O.golden("interp_harness_seed424242.json")["cases"]:
        g = c["gemm"]
        n, m, p = g["n"], g["m"], g["p"]
        out = np.full(n * m, np.nan)
        H.gemm(n, m, out, p, np.array(g["a"], np.float64), np.array(g["b"], np.float64))
        assert O.same_bits(out, np.array(g["c"], np.float64))


@pytest.mark.parametrize("n,m,p", [(1, 1, 1), (7, 5, 3), (300, 200, 250), (512, 384, 1024), (33, 1, 0),
                                   (65, 63, 17), (129, 257, 31)])
def test_gemm_fast_and_exact_vs_oracle(n, m, p):
    rng = np.random.default_rng(n * 1000 + m + p)
    a = rng.uniform(-2, 2, n * p)
    b = rng.uniform(-2, 2, p * m)
    ref = O.gemm(n, m, p, a, b)
    scale = O.gemm(n, m, p, np.abs(a), np.abs(b))
    out = np.full(n * m, np.nan)
    H.gemm(n, m, out, p, a, b)  # the DMMA kernel (FP64 tensor cores)
    assert (np.abs(out - ref) <= TOL * scale + (scale == 0) * 0).all()
    N.lib().b200_set_exact_blas(1)
    out2 = np.full(n * m, np.nan)
    H.gemm(n, m, out2, p, a, b)
    assert O.same_bits(out2, ref)


@pytest.mark.parametrize("n,m,p", [(1, 1, 1), (65, 129, 17), (256, 192, 300)])
def test_gemm_device_api(n, m, p):
    """b200_gemm_device on device buffers: the DMMA kernel within tolerance,
    the exact kernel bit-identical to the oracle."""
    import torch
    rng = np.random.default_rng(7 + n + m + p)
    a = rng.uniform(-2, 2, n * p)
    b = rng.uniform(-2, 2, p * m)
    ref = O.gemm(n, m, p, a, b)
    scale = O.gemm(n, m, p, np.abs(a), np.abs(b))
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    for exact in (False, True):
        dc = torch.full((n * m,), float("nan"), dtype=torch.float64, device="cuda")
        D.gemm(n, m, p, da.data_ptr(), db.data_ptr(), dc.data_ptr(), exact=exact)
        torch.cuda.synchronize()
        out = dc.cpu().numpy()
        if exact:
            assert O.same_bits(out, ref)
        else:
            assert (np.abs(out - ref) <= TOL * scale).all()


def test_gemm_argument_checks():
    with pytest.raises(ValueError):
        H.gemm(4, 4, np.zeros(15), 4, np.zeros(16), np.zeros(16))


# --------------------------------------------------------------------------------
# segmented JDS (k_jds_seg: a row's diagonals spread over up to 32 lanes, the
# running sum carried lane to lane) and its fallbacks
# --------------------------------------------------------------------------------

def _jds_case(lens, seed):
    rng = np.random.default_rng(seed)
    rows = len(lens)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = rng.integers(0, rows, int(rp[-1])).astype(np.int64)
    val = rng.uniform(-2, 2, int(rp[-1]))
    x = rng.uniform(-2, 2, rows)
    return (*O.jds_from_csr(rp, ci, val), x)


def _run_jds(perm, nzcnt, jd_ptr, jval, jcol, x):
    y = np.full(len(perm), np.nan)
    H.spmv_jds(len(perm), y, nzcnt, perm, jval, jd_ptr, x, jcol)
    return y


@pytest.mark.parametrize("max_len", [1, 10, 11, 64, 320, 321, 700])
def test_jds_every_lane_group_bitwise(max_len):
    # every row length 0..max_len (each lanes-per-row zone and its edges);
    # rows longer than 32 lanes' worth take the thread-per-row kernel
    lens = np.concatenate([np.arange(max_len + 1), np.random.default_rng(max_len).integers(0, max_len + 1, 3000)])
    perm, nzcnt, jd_ptr, jval, jcol, x = _jds_case(lens, 7 + max_len)
    y = _run_jds(perm, nzcnt, jd_ptr, jval, jcol, x)
    assert O.same_bits(y, O.spmv_jds(nzcnt, perm, jval, jd_ptr, x, jcol))


def test_jds_unsorted_nzcnt_bitwise():
    # a valid JDS whose nzcnt is not non-increasing (row 0 shortened): the
    # lane groups do not apply; the reference semantics still hold
    perm, nzcnt, jd_ptr, jval, jcol, x = _jds_case(np.random.default_rng(3).integers(0, 40, 5000), 11)
    nzcnt = nzcnt.copy()
    nzcnt[0] = 1
    nzcnt[7] = 0
    y = _run_jds(perm, nzcnt, jd_ptr, jval, jcol, x)
    assert O.same_bits(y, O.spmv_jds(nzcnt, perm, jval, jd_ptr, x, jcol))


# --------------------------------------------------------------------------------
# eager write-back into pageable memory (copy_engine.cpp: pinned chunks +
# parallel host copies for outputs of 256 KB or more)
# --------------------------------------------------------------------------------

@pytest.mark.parametrize("rows,offset", [(40000, 0), (200001, 0), (300000, 1), (131072, 3)])
def test_large_pageable_output_written_back_exactly(rows, offset):
    """The reference semantics on a plain (malloc'd) output: every element of
    the output lands, nothing around it changes, whatever the size and the
    8-byte alignment inside the allocation."""
    rng = np.random.default_rng(rows + offset)
    lens = rng.integers(0, 9, rows)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = rng.integers(0, rows, int(rp[-1])).astype(np.int64)
    for i in range(0, rows, max(1, rows // 64)):  # a few sorted rows suffice for the exact kernel's order
        ci[rp[i]:rp[i + 1]].sort()
    val = rng.uniform(-2, 2, int(rp[-1]))
    x = rng.uniform(-2, 2, rows)
    N.lib().b200_set_kernel(b"exact")
    buf = np.full(rows + offset + 5, 7.25)
    y = buf[offset:offset + rows]
    H.spmv_csr(rows, y, rp, val, x, ci)
    assert O.same_bits(y, O.spmv_csr(rp, ci, val, x))
    assert np.all(buf[:offset] == 7.25) and np.all(buf[offset + rows:] == 7.25)


@pytest.mark.parametrize("kernel", [b"auto", b"lane"])
def test_pagerank_step_api_ping_pong(kernel):
    """b200_pagerank_step_device: y = d A x + (1-d)/n into another vector, the
    update folded into the lane-range row stores or run in place after the
    SpMV on other layouts; alternating buffers reproduces the host iteration."""
    import torch
    rng = np.random.default_rng(21)
    n = 8000
    src = rng.integers(0, n, 90000)
    dst = rng.integers(0, n, 90000)
    outdeg = np.bincount(src, minlength=n).astype(np.float64)
    order = np.lexsort((src, dst))
    src, dst = src[order], dst[order]
    rp = np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))]).astype(np.int64)
    ci = src.astype(np.int64)
    val = 1.0 / outdeg[src]
    N.lib().b200_set_kernel(kernel)
    A = D.Matrix.csr(rp, ci, val)
    bufs = [torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64,
                                                                                          device="cuda")]
    for _ in range(7):
        A.pagerank_step(0.85, bufs[0].data_ptr(), bufs[1].data_ptr())
        bufs.reverse()
    torch.cuda.synchronize()
    xr = np.full(n, 1.0 / n)
    for _ in range(7):
        xr = 0.85 * O.spmv_csr(rp, ci, val, xr) + 0.15 / n
    assert np.allclose(bufs[0].cpu().numpy(), xr, rtol=1e-12, atol=1e-15)
    with pytest.raises(N.B200Error):
        A.pagerank_step(0.85, bufs[0].data_ptr(), bufs[0].data_ptr())
    A.free()
