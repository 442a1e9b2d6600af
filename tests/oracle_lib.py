"""ctypes bindings for the test-only oracle libraries.

* ``oracle/liboracle.so`` — the C restatement (oracle/oracle.c), built by
  ``make -C oracle`` (here or on the GPU box: it only needs gcc).
* ``oracle/_ref/liblilac_ref.so`` — the reference's own sources compiled in
  place plus oracle/ref_shim.cpp; present only where /root/reference was
  available at build time (travels to the GPU box as a built file).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")

i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
I64 = C.c_int64


def ptr(a: np.ndarray):
    if a.dtype == np.int64:
        return a.ctypes.data_as(i64p)
    if a.dtype == np.float64:
        return a.ctypes.data_as(f64p)
    return C.c_void_p(a.ctypes.data)


_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is not None:
        return _oracle
    so = os.path.join(ORACLE_DIR, "liboracle.so")
    src = os.path.join(ORACLE_DIR, "oracle.c")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR, "all"], check=True)
    L = C.CDLL(so)
    L.orc_spmv_csr.argtypes = [I64, f64p, i64p, f64p, f64p, i64p, I64, I64]
    L.orc_spmv_csr.restype = C.c_int
    L.orc_spmv_jds.argtypes = [I64, f64p, i64p, i64p, f64p, i64p, f64p, i64p, I64, I64, I64]
    L.orc_spmv_jds.restype = C.c_int
    L.orc_dot.argtypes = [f64p, I64, f64p, f64p]
    L.orc_gemm.argtypes = [I64, I64, f64p, I64, f64p, f64p]
    L.orc_axpy.argtypes = [I64, f64p, C.c_double, f64p]
    L.orc_spmv_csr_mt.argtypes = [I64, f64p, i64p, f64p, f64p, i64p, C.c_int]
    L.orc_count_nonzeros.argtypes = [I64, I64, f64p]
    L.orc_count_nonzeros.restype = I64
    L.orc_csr_from_dense.argtypes = [I64, I64, f64p, f64p, i64p, i64p]
    L.orc_csr_max_row.argtypes = [I64, i64p]
    L.orc_csr_max_row.restype = I64
    L.orc_jds_from_csr.argtypes = [I64, i64p, f64p, i64p, i64p, i64p, i64p, f64p, i64p]
    L.orc_fnv1a.argtypes = [C.c_void_p, C.c_size_t]
    L.orc_fnv1a.restype = C.c_uint64
    L.orc_partition_rows.argtypes = [I64, i64p, C.c_int, i64p]
    L.orc_npb_makea.argtypes = [I64, C.c_int, C.c_double, i64p, i64p, f64p, i64p]
    L.orc_npb_makea.restype = C.c_int
    L.orc_npb_cg.argtypes = [I64, i64p, i64p, f64p, C.c_int, C.c_double, f64p]
    L.orc_npb_cg.restype = C.c_double
    L.orc_npb_outer.argtypes = [I64, i64p, i64p, f64p, f64p, f64p, f64p, f64p, f64p, C.c_double, C.c_int, f64p]
    L.orc_npb_outer.restype = C.c_double
    L.orc_spmv_jds_mt.argtypes = [I64, f64p, i64p, i64p, f64p, i64p, f64p, i64p, C.c_int]
    _oracle = L
    return L


def ref_available() -> bool:
    return os.path.exists(os.path.join(ORACLE_DIR, "_ref", "liblilac_ref.so"))


def ref() -> C.CDLL:
    """The reference's own CPU harness (oracle/_ref)."""
    global _ref
    if _ref is not None:
        return _ref
    L = C.CDLL(os.path.join(ORACLE_DIR, "_ref", "liblilac_ref.so"))
    L.ref_prepare_csr.argtypes = [I64, i64p, f64p, f64p, i64p, I64, I64]
    L.ref_prepare_csr.restype = C.c_void_p
    L.ref_prepare_jds.argtypes = [I64, i64p, i64p, f64p, i64p, f64p, i64p, I64, I64, I64]
    L.ref_prepare_jds.restype = C.c_void_p
    L.ref_prepare_dot.argtypes = [I64, f64p, f64p]
    L.ref_prepare_dot.restype = C.c_void_p
    L.ref_call.argtypes = [C.c_void_p]
    L.ref_call.restype = C.c_int
    L.ref_output.argtypes = [C.c_void_p, f64p]
    L.ref_free.argtypes = [C.c_void_p]
    L.ref_set_floats.argtypes = [C.c_void_p, C.c_int, f64p, I64]
    L.ref_set_floats.restype = C.c_int
    L.ref_scalar.argtypes = [C.c_void_p]
    L.ref_scalar.restype = C.c_double
    L.ref_last_error.restype = C.c_char_p
    L.ref_infer_interface.argtypes = [C.c_char_p, C.c_char_p, I64]
    L.ref_infer_interface.restype = C.c_int
    L.ref_gen_harness.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, I64]
    L.ref_gen_harness.restype = I64
    L.ref_fnv1a.argtypes = [C.c_void_p, C.c_size_t]
    L.ref_fnv1a.restype = C.c_uint64
    _ref = L
    return L


# --------------------------------------------------------------------------
# convenience wrappers
# --------------------------------------------------------------------------

def spmv_csr(row_ptr, col_ind, val, x, rows=None):
    rows = len(row_ptr) - 1 if rows is None else rows
    y = np.zeros(rows, dtype=np.float64)
    rc = oracle().orc_spmv_csr(rows, ptr(y), ptr(row_ptr), ptr(val), ptr(x), ptr(col_ind),
                               len(val), len(x))
    if rc != 0:
        raise IndexError("OutOfBounds")
    return y


def spmv_csr_mt(row_ptr, col_ind, val, x, nthreads=0):
    rows = len(row_ptr) - 1
    y = np.zeros(rows, dtype=np.float64)
    oracle().orc_spmv_csr_mt(rows, ptr(y), ptr(row_ptr), ptr(val), ptr(x), ptr(col_ind), nthreads)
    return y


def spmv_jds(nzcnt, perm, val, jd_ptr, x, col_ind):
    rows = len(perm)
    y = np.zeros(rows, dtype=np.float64)
    rc = oracle().orc_spmv_jds(rows, ptr(y), ptr(nzcnt), ptr(perm), ptr(val), ptr(jd_ptr), ptr(x),
                               ptr(col_ind), len(val), len(jd_ptr), len(x))
    if rc != 0:
        raise IndexError("OutOfBounds")
    return y


def dot(a, b):
    r = np.zeros(1, dtype=np.float64)
    oracle().orc_dot(ptr(r), len(a), ptr(a), ptr(b))
    return r[0]


def gemm(n, m, p, a, b):
    """c (n x m) = a (n x p) b (p x m), row-major, the reference's k order."""
    c = np.zeros(n * m, dtype=np.float64)
    oracle().orc_gemm(n, m, ptr(c), p, ptr(np.ascontiguousarray(a, np.float64).ravel()),
                      ptr(np.ascontiguousarray(b, np.float64).ravel()))
    return c


def axpy(y, alpha, x):
    y = y.copy()
    oracle().orc_axpy(len(y), ptr(y), alpha, ptr(x))
    return y


def csr_from_dense(dense: np.ndarray):
    rows, cols = dense.shape
    d = np.ascontiguousarray(dense, dtype=np.float64)
    nnz = oracle().orc_count_nonzeros(rows, cols, ptr(d))
    val = np.zeros(nnz, np.float64)
    ci = np.zeros(nnz, np.int64)
    rp = np.zeros(rows + 1, np.int64)
    oracle().orc_csr_from_dense(rows, cols, ptr(d), ptr(val), ptr(ci), ptr(rp))
    return rp, ci, val


def jds_from_csr(row_ptr, col_ind, val):
    rows = len(row_ptr) - 1
    max_nz = oracle().orc_csr_max_row(rows, ptr(row_ptr))
    perm = np.zeros(rows, np.int64)
    nzcnt = np.zeros(rows, np.int64)
    jd_ptr = np.zeros(max_nz + 1, np.int64)
    jval = np.zeros(len(val), np.float64)
    jcol = np.zeros(len(val), np.int64)
    oracle().orc_jds_from_csr(rows, ptr(row_ptr), ptr(val), ptr(col_ind), ptr(perm), ptr(nzcnt),
                              ptr(jd_ptr), ptr(jval), ptr(jcol))
    return perm, nzcnt, jd_ptr, jval, jcol


def partition_rows(row_ptr, k):
    rows = len(row_ptr) - 1
    b = np.zeros(k + 1, np.int64)
    oracle().orc_partition_rows(rows, ptr(row_ptr), k, ptr(b))
    return b


def npb_makea(na, nonzer, shift):
    rp = np.zeros(na + 1, np.int64)
    nnz = np.zeros(1, np.int64)
    assert oracle().orc_npb_makea(na, nonzer, shift, ptr(rp), None, None, ptr(nnz)) == 0
    ci = np.zeros(nnz[0], np.int64)
    val = np.zeros(nnz[0], np.float64)
    assert oracle().orc_npb_makea(na, nonzer, shift, ptr(rp), ptr(ci), ptr(val), ptr(nnz)) == 0
    return rp, ci, val


def npb_cg(row_ptr, col_ind, val, niter, shift):
    rn = np.zeros(1, np.float64)
    z = oracle().orc_npb_cg(len(row_ptr) - 1, ptr(row_ptr), ptr(col_ind), ptr(val), niter, shift,
                            ptr(rn))
    return z, rn[0]


class NpbOuter:
    """NPB outer iterations of the C restatement from a caller-held x (x = 1
    initially), SpMV on `nthreads` host threads (0 = all): the native CPU
    baseline of bench.py and the zeta checker of its e2e leg."""

    def __init__(self, row_ptr, col_ind, val, shift, nthreads=0):
        self.rp, self.ci, self.val, self.shift, self.nthreads = row_ptr, col_ind, val, shift, nthreads
        n = len(row_ptr) - 1
        self.n = n
        self.x = np.ones(n)
        self.work = [np.zeros(n) for _ in range(4)]

    def step(self):
        rn = np.zeros(1)
        z, p, q, r = self.work
        zeta = oracle().orc_npb_outer(self.n, ptr(self.rp), ptr(self.ci), ptr(self.val), ptr(self.x), ptr(z),
                                      ptr(p), ptr(q), ptr(r), self.shift, self.nthreads, ptr(rn))
        return zeta, rn[0]


def spmv_jds_mt(nzcnt, perm, val, jd_ptr, x, col_ind, nthreads=0):
    rows = len(perm)
    y = np.zeros(rows, dtype=np.float64)
    oracle().orc_spmv_jds_mt(rows, ptr(y), ptr(nzcnt), ptr(perm), ptr(val), ptr(jd_ptr), ptr(x), ptr(col_ind),
                             nthreads)
    return y


def fnv1a(b: bytes) -> int:
    buf = C.create_string_buffer(b, len(b))
    return oracle().orc_fnv1a(buf, len(b))


# --------------------------------------------------------------------------
# golden fixtures
# --------------------------------------------------------------------------

def golden(name: str):
    with open(os.path.join(GOLDEN_DIR, name)) as f:
        return json.load(f)


def case_arrays(c):
    """numpy views of one golden case (tests/golden/*.json)."""
    out = {
        "rows": c["rows"],
        "cols": c["cols"],
        "dense": np.array(c["dense"], np.float64).reshape(c["rows"], c["cols"]),
        "x": np.array(c["x"], np.float64),
        "row_ptr": np.array(c["csr"]["row_ptr"], np.int64),
        "col_ind": np.array(c["csr"]["col_ind"], np.int64),
        "val": np.array(c["csr"]["val"], np.float64),
        "perm": np.array(c["jds"]["perm"], np.int64),
        "nzcnt": np.array(c["jds"]["nzcnt"], np.int64),
        "jd_ptr": np.array(c["jds"]["jd_ptr"], np.int64),
        "jds_col_ind": np.array(c["jds"]["col_ind"], np.int64),
        "jds_val": np.array(c["jds"]["val"], np.float64),
        "y_csr": np.array(c["y_csr"], np.float64),
        "y_jds": np.array(c["y_jds"], np.float64),
        "y_dense": np.array(c["y_dense"], np.float64),
    }
    return out


def all_golden_cases():
    cases = []
    s5 = golden("sample5.json")
    cases.append(("sample5.ones", s5["ones"]))
    cases.append(("sample5.counting", s5["counting"]))
    for fn in ("what_csr_seed20240817.json", "what_jds_seed7.json", "interp_harness_seed424242.json"):
        for i, c in enumerate(golden(fn)["cases"]):
            cases.append((f"{fn}[{i}]", c))
    return cases


def same_bits(a: np.ndarray, b: np.ndarray) -> bool:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


# --------------------------------------------------------------------------
# the reference's own CPU harness driven by a host loop (bench.py's reference
# arm and the class A zeta test): stock "lilac.spmv_csr" / "lilac.spmv_jds" /
# "lilac.dotproduct" HarnessFns (interp.cpp:330-389), one prepared call per
# host thread on an nnz-balanced slice, run concurrently (ctypes releases the
# GIL; the interpreter has no shared mutable state)
# --------------------------------------------------------------------------

def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def _run_parallel(fns):
    import threading
    if len(fns) == 1:
        fns[0]()
        return
    th = [threading.Thread(target=f) for f in fns]
    for t in th:
        t.start()
    for t in th:
        t.join()


class RefCsr:
    """y = A x through `lilac.spmv_csr`, rows cut into T nnz-balanced slices."""

    def __init__(self, row_ptr, col_ind, val, ncols, threads=None, rows=None):
        R = ref()
        self.R = R
        self.rows = len(row_ptr) - 1 if rows is None else rows
        T = max(1, min(threads or host_threads(), max(1, self.rows)))
        rp = row_ptr
        nnz = int(rp[self.rows] - rp[0])
        b = [0]
        for t in range(1, T):
            b.append(max(b[-1], int(np.searchsorted(rp[: self.rows + 1], rp[0] + nnz * t // T))))
        b.append(self.rows)
        self.bounds = b
        self.ncols = ncols
        self.h = []
        x0 = np.zeros(max(ncols, 1))
        for t in range(T):
            r0, r1 = b[t], b[t + 1]
            a, e = int(rp[r0]), int(rp[r1])
            rpt = np.ascontiguousarray(rp[r0:r1 + 1] - rp[r0])
            cit = np.ascontiguousarray(col_ind[a:e])
            vt = np.ascontiguousarray(val[a:e])
            self.h.append(R.ref_prepare_csr(r1 - r0, ptr(rpt), ptr(vt), ptr(x0), ptr(cit), e - a, ncols))

    def __call__(self, x, y):
        R = self.R

        def job(t):
            def f():
                R.ref_set_floats(self.h[t], 4, ptr(x), self.ncols)
                if R.ref_call(self.h[t]) != 0:
                    raise IndexError(R.ref_last_error().decode())
                R.ref_output(self.h[t], ptr(y[self.bounds[t]:self.bounds[t + 1]]))
            return f
        _run_parallel([job(t) for t in range(len(self.h))])
        return y

    def free(self):
        for h in self.h:
            self.R.ref_free(h)
        self.h = []


class RefDot:
    """a . b through `lilac.dotproduct` on T element slices; the slice partials
    are summed in slice order."""

    def __init__(self, n, threads=None):
        R = ref()
        self.R = R
        T = max(1, min(threads or host_threads(), max(1, n // 4096)))
        self.bounds = [n * t // T for t in range(T + 1)]
        z = np.zeros(max(n, 1))
        self.h = [R.ref_prepare_dot(self.bounds[t + 1] - self.bounds[t], ptr(z), ptr(z)) for t in range(T)]

    def __call__(self, a, b):
        R = self.R
        out = [0.0] * len(self.h)

        def job(t):
            def f():
                lo, hi = self.bounds[t], self.bounds[t + 1]
                R.ref_set_floats(self.h[t], 1, ptr(a[lo:hi]), hi - lo)
                R.ref_set_floats(self.h[t], 2, ptr(b[lo:hi]), hi - lo)
                R.ref_call(self.h[t])
                out[t] = R.ref_scalar(self.h[t])
            return f
        _run_parallel([job(t) for t in range(len(self.h))])
        s = 0.0
        for v in out:
            s += v
        return s

    def free(self):
        for h in self.h:
            self.R.ref_free(h)
        self.h = []


class RefNpbCG:
    """NPB CG outer iterations whose SpMVs and dot products are the reference's
    HarnessFns (RefCsr / RefDot) and whose vector updates are host loops
    (numpy): a LiLAC-rewritten NPB CG linked against the reference CPU harness
    (SURVEY §8(d) input 1). x starts at 1."""

    def __init__(self, row_ptr, col_ind, val, shift, threads=None):
        n = len(row_ptr) - 1
        self.n, self.shift = n, shift
        self.spmv = RefCsr(row_ptr, col_ind, val, n, threads)
        self.dot = RefDot(n, threads)
        self.x = np.ones(n)
        self.z, self.p, self.q, self.r = (np.zeros(n) for _ in range(4))
        self.spmvs = self.dots = 0

    def step(self, cgitmax=25):
        x, z, p, q, r = self.x, self.z, self.p, self.q, self.r
        z[:] = 0.0
        q[:] = 0.0
        r[:] = x
        p[:] = r
        rho = self.dot(r, r)
        for _ in range(cgitmax):
            self.spmv(p, q)
            d = self.dot(p, q)
            alpha = rho / d
            rho0 = rho
            z += alpha * p
            r -= alpha * q
            rho = self.dot(r, r)
            beta = rho / rho0
            p *= beta
            p += r
        self.spmv(z, r)
        res = x - r
        rnorm = float(np.sqrt(self.dot(res, res)))
        t1 = self.dot(x, z)
        t2 = 1.0 / np.sqrt(self.dot(z, z))
        x[:] = t2 * z
        self.spmvs += cgitmax + 1
        self.dots += 2 * cgitmax + 4
        return self.shift + 1.0 / t1, rnorm

    def free(self):
        self.spmv.free()
        self.dot.free()
