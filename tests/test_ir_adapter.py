"""IR-pipeline adapter: the B200 harnesses registered in the
reference's interp::HarnessRegistry (paper_2001_07938_b200/adapters/
interp_b200.cpp), driven through the reference's own parse → detect →
rewrite → interp::run flow (oracle/ir_shim.cpp over oracle/_ref).

The bar, as the reference's pipeline test (test_cli.cpp:156-168): the
rewritten module run with the harness must produce exactly what the original
module's interpretation produces. CPU tests pin the shim and the IR inputs
with the reference's own harness; GPU tests swap in the B200 registry."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle_lib as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "oracle", "_ref", "liblilac_ir_b200.so")
IRDIR = os.path.join(ROOT, "tests", "golden", "ir")

# the reference's kernels.lilac computations (fixtures/lilac/kernels.lilac:1-19)
SPEC = b"""
COMPUTATION spmv_csr
forall (0 <= i < rows) {
    output[i] = dot (row_ptr[i] <= j < row_ptr[i + 1]) val[j] * x[col_ind[j]];
}

COMPUTATION dotproduct
result = dot (0 <= i < length) a[i] * b[i];

COMPUTATION spmv_jds
forall (0 <= i < rows) {
    output[i] = dot (0 <= k < nzcnt[perm[i]]) val[jd_ptr[k] + perm[i]] * x[col_ind[jd_ptr[k] + perm[i]]];
}

COMPUTATION gemm
forall (0 <= i < n) {
    forall (0 <= j < m) {
        c[i * m + j] = dot (0 <= k < p) a[i * p + k] * b[k * m + j];
    }
}
"""

NONE, REFERENCE, B200 = 0, 1, 2

pytestmark = pytest.mark.skipif(not os.path.exists(SHIM), reason="oracle/_ref/liblilac_ir_b200.so not built")


def shim():
    L = C.CDLL(SHIM)
    L.ir_open.restype = C.c_void_p
    L.ir_open.argtypes = [C.c_char_p]
    L.ir_close.argtypes = [C.c_void_p]
    L.ir_error.restype = C.c_char_p
    L.ir_rewrite.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p]
    L.ir_text.restype = C.c_int64
    L.ir_text.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_int64]
    L.ir_add_i64.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64]
    L.ir_add_f64.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64]
    L.ir_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.c_char_p, C.c_void_p, C.c_void_p, C.c_int,
                         C.POINTER(C.c_double)]
    L.ir_call_harness.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_char_p, C.c_void_p, C.c_void_p, C.c_int,
                                  C.POINTER(C.c_double)]
    L.ir_read_f64.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
    L.ir_write_version.restype = C.c_uint64
    L.ir_write_version.argtypes = [C.c_void_p, C.c_int]
    return L


class Session:
    """One parsed module plus a base memory image (interp::Memory buffers)."""

    def __init__(self, lir_name, what=None):
        self.L = shim()
        with open(os.path.join(IRDIR, lir_name), "rb") as f:
            self.h = self.L.ir_open(f.read())
        assert self.h, self.L.ir_error()
        self.applied = self.L.ir_rewrite(self.h, SPEC, what.encode()) if what else 0
        assert self.applied >= 0, self.L.ir_error()
        self.args = []

    def text(self, rewritten):
        n = self.L.ir_text(self.h, rewritten, None, 0)
        buf = C.create_string_buffer(n + 1)
        self.L.ir_text(self.h, rewritten, buf, n + 1)
        return buf.value.decode()

    def scalar(self, v):
        self.args.append((0, int(v)))

    def ints(self, label, a):
        a = np.ascontiguousarray(a, np.int64)
        b = self.L.ir_add_i64(self.h, label.encode(), a.ctypes.data, len(a))
        assert b >= 0, self.L.ir_error()
        self.args.append((1, b))
        return b

    def floats(self, label, a):
        a = np.ascontiguousarray(a, np.float64)
        b = self.L.ir_add_f64(self.h, label.encode(), a.ctypes.data, len(a))
        assert b >= 0, self.L.ir_error()
        self.args.append((1, b))
        return b

    def _argv(self):
        kinds = np.array([k for k, _ in self.args], np.int32)
        vals = np.array([v for _, v in self.args], np.int64)
        return kinds, vals

    def run(self, rewritten, backend, entry):
        kinds, vals = self._argv()
        ret = C.c_double(np.nan)
        rc = self.L.ir_run(self.h, rewritten, backend, SPEC, entry.encode(), kinds.ctypes.data, vals.ctypes.data,
                           len(kinds), C.byref(ret))
        if rc != 0:
            raise RuntimeError(self.L.ir_error().decode())
        return ret.value

    def call(self, backend, name):
        kinds, vals = self._argv()
        ret = C.c_double(np.nan)
        rc = self.L.ir_call_harness(self.h, backend, SPEC, name.encode(), kinds.ctypes.data, vals.ctypes.data,
                                    len(kinds), C.byref(ret))
        if rc != 0:
            raise RuntimeError(self.L.ir_error().decode())
        return ret.value

    def read(self, buf, n):
        out = np.empty(n)
        assert self.L.ir_read_f64(self.h, buf, out.ctypes.data, n) == 0, self.L.ir_error()
        return out

    def version(self, buf):
        return self.L.ir_write_version(self.h, buf)

    def close(self):
        self.L.ir_close(self.h)


def csr_session(rp, ci, val, x, rows=None):
    rows = len(rp) - 1 if rows is None else rows
    s = Session("spmv_rows.lir", "spmv_csr")
    s.scalar(rows)
    out = s.floats("y", np.zeros(max(rows, 1)))
    s.ints("rp", rp)
    s.floats("a", val)
    s.floats("v", x)
    s.ints("c", ci)
    return s, out, rows


def sample5():
    g = O.golden("sample5.json")
    c = O.case_arrays(g["ones"])
    xs = {"ones": c["x"], "counting": O.case_arrays(g["counting"])["x"]}
    ys = {"ones": c["y_csr"], "counting": O.case_arrays(g["counting"])["y_csr"]}
    return c["row_ptr"], c["col_ind"], c["val"], (xs, ys)


def rand_csr(rows, cols, per_row, seed):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 2 * per_row + 1, rows)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = rng.integers(0, cols, int(rp[-1])).astype(np.int64)
    val = rng.uniform(-2, 2, int(rp[-1]))
    return rp, ci, val


# ---- CPU: the pipeline and the shim, with the reference's own harness -----------

def test_inputs_are_rewritten_to_harness_calls():
    s = Session("spmv_rows.lir", "spmv_csr")
    assert s.applied == 1
    assert "call @lilac.spmv_csr(%n, %y, %rp, %a, %v, %c)" in s.text(1)
    d = Session("dot_loop.lir", "dotproduct")
    assert d.applied == 1
    assert "call @lilac.dotproduct(%len, %u, %w)" in d.text(1)


def test_reference_harness_reproduces_the_original_module():
    rp, ci, val, (xs, ys) = sample5()
    for name in ("ones", "counting"):
        s, out, rows = csr_session(rp, ci, val, xs[name])
        s.run(0, NONE, "csr_rows")
        y0 = s.read(out, rows)
        s.run(1, REFERENCE, "csr_rows")
        y1 = s.read(out, rows)
        assert np.array_equal(y0, ys[name])
        assert y1.tobytes() == y0.tobytes()
        s.close()


def gemm_session(n, m, p, seed):
    rng = np.random.default_rng(seed)
    s = Session("gemm_loops.lir", "gemm")
    s.scalar(n)
    s.scalar(m)
    out = s.floats("out", np.zeros(max(n * m, 1)))
    s.scalar(p)
    s.floats("L", rng.uniform(-2, 2, max(n * p, 1)))
    s.floats("R", rng.uniform(-2, 2, max(p * m, 1)))
    return s, out


def test_gemm_loops_rewritten_and_reproduced_by_the_reference_harness():
    s, out = gemm_session(9, 7, 5, 1)
    assert s.applied == 1
    assert "call @lilac.gemm(%rows, %cols, %out, %inner, %L, %R)" in s.text(1)
    s.run(0, NONE, "matmul")
    y0 = s.read(out, 63)
    s.run(1, REFERENCE, "matmul")
    assert s.read(out, 63).tobytes() == y0.tobytes()


def test_rewritten_module_needs_a_registered_harness():
    rp, ci, val, _ = sample5()
    s, _, _ = csr_session(rp, ci, val, np.ones(5))
    with pytest.raises(RuntimeError, match="UnregisteredHarness|lilac.spmv_csr"):
        s.run(1, NONE, "csr_rows")


# ---- GPU: the B200 registry behind the same pipeline -------------------------------

@pytest.fixture
def exact_kernels():
    from paper_2001_07938_b200 import _native as N
    L = N.lib()
    L.b200_set_kernel(b"exact")
    L.b200_set_exact_blas(1)
    yield
    L.b200_set_kernel(b"auto")
    L.b200_set_exact_blas(0)


@pytest.mark.gpu
def test_b200_registry_reproduces_sample5_through_the_pipeline():
    rp, ci, val, (xs, ys) = sample5()
    for name in ("ones", "counting"):
        s, out, rows = csr_session(rp, ci, val, xs[name])
        s.run(0, NONE, "csr_rows")
        y0 = s.read(out, rows)
        v0 = s.version(out)
        s.run(1, B200, "csr_rows")
        y1 = s.read(out, rows)
        assert y1.tobytes() == y0.tobytes() == ys[name].tobytes()
        assert s.version(out) == v0  # one store per output element, as the interpreter
        s.close()


@pytest.mark.gpu
def test_b200_registry_bit_identical_with_exact_kernels(exact_kernels):
    rp, ci, val = rand_csr(3000, 2500, 9, 424242)
    x = np.random.default_rng(1).uniform(-2, 2, 2500)
    s, out, rows = csr_session(rp, ci, val, x)
    s.run(0, NONE, "csr_rows")
    y0 = s.read(out, rows)
    s.run(1, B200, "csr_rows")
    assert s.read(out, rows).tobytes() == y0.tobytes()
    d = Session("dot_loop.lir", "dotproduct")
    d.scalar(2500)
    d.floats("u", x)
    d.floats("w", x[::-1].copy())
    r0 = d.run(0, NONE, "inner")
    r1 = d.run(1, B200, "inner")
    assert np.float64(r1).tobytes() == np.float64(r0).tobytes()


@pytest.mark.gpu
def test_b200_registry_fast_kernels_within_tolerance():
    rp, ci, val = rand_csr(200_000, 200_000, 12, 99)
    x = np.random.default_rng(2).uniform(-2, 2, 200_000)
    s, out, rows = csr_session(rp, ci, val, x)
    s.run(0, NONE, "csr_rows")
    y0 = s.read(out, rows)
    s.run(1, B200, "csr_rows")
    y1 = s.read(out, rows)
    scale = O.spmv_csr(rp, ci, np.abs(val), np.abs(x), rows)
    assert (np.abs(y1 - y0) <= 1e-12 * scale).all()


@pytest.mark.gpu
def test_b200_jds_harness_bit_identical_to_reference_harness():
    rp, ci, val = rand_csr(4000, 3000, 7, 7)
    x = np.random.default_rng(3).uniform(-2, 2, 3000)
    perm, nzcnt, jd_ptr, jval, jcol = O.jds_from_csr(rp, ci, val)
    jd = {"perm": perm, "nzcnt": nzcnt, "jd_ptr": jd_ptr, "val": jval, "col_ind": jcol}
    outs = []
    for backend in (REFERENCE, B200):
        s = Session("dot_loop.lir")  # any module: the harness is called directly
        s.scalar(4000)
        out = s.floats("output", np.zeros(4000))
        s.ints("nzcnt", jd["nzcnt"])
        s.ints("perm", jd["perm"])
        s.floats("val", jd["val"])
        s.ints("jd_ptr", jd["jd_ptr"])
        s.floats("x", x)
        s.ints("col_ind", jd["col_ind"])
        s.call(backend, "lilac.spmv_jds")
        outs.append(s.read(out, 4000))
    assert outs[1].tobytes() == outs[0].tobytes()


@pytest.mark.gpu
def test_b200_registry_raises_out_of_bounds_like_the_reference():
    rp, ci, val, _ = sample5()
    for backend in (REFERENCE, B200):
        s, out, rows = csr_session(rp, ci, val, np.ones(3))  # x too short for column 4
        with pytest.raises(RuntimeError, match="OutOfBounds"):
            s.run(1, backend, "csr_rows")
        s.close()


@pytest.mark.gpu
def test_b200_registry_gemm_through_the_pipeline(exact_kernels):
    s, out = gemm_session(40, 33, 27, 2)
    s.run(0, NONE, "matmul")
    y0 = s.read(out, 40 * 33)
    s.run(1, B200, "matmul")
    assert s.read(out, 40 * 33).tobytes() == y0.tobytes()


@pytest.mark.gpu
def test_b200_registry_gemm_fast_path_within_tolerance():
    n, m, p = 64, 48, 80
    s, out = gemm_session(n, m, p, 3)
    s.run(0, NONE, "matmul")
    y0 = s.read(out, n * m)
    s.run(1, B200, "matmul")
    y1 = s.read(out, n * m)
    assert np.allclose(y1, y0, rtol=0, atol=1e-12 * 4 * p)
