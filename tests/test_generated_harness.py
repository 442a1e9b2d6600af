"""the drop-in behind the reference's plugin API.

paper_2001_07938_b200/specs/b200.lilac is a LiLAC-How spec for this backend.
The reference's own generator (harnessgen::gen_all, via oracle/_ref) turns it
into tests/golden/b200gen_spmv_csr.gen.cpp, which build.py compiles UNCHANGED
against include/lilac/marshal.hpp into liblilac_b200_gen.so. (The reference's
own golden cuSPARSE TU does not compile against its own header: SURVEY §8(b)
B7.) The generated entry point must behave like every other spmv_csr harness.
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle_lib as O

GEN_LIB = os.path.join(O.ROOT, "paper_2001_07938_b200", "liblilac_b200_gen.so")


@pytest.mark.skipif(not O.ref_available(), reason="needs oracle/_ref (the reference's generator)")
def test_generated_harness_is_what_the_reference_generator_emits():
    r = subprocess.run([sys.executable, os.path.join(O.ROOT, "tools", "gen_b200_harness.py"), "--check"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_generated_harness_compiled_and_exports_the_harness_symbol():
    from paper_2001_07938_b200 import build as B
    B.build_generated_harness()
    L = C.CDLL(GEN_LIB)
    assert hasattr(L, "b200gen_spmv_csr")
    src = open(os.path.join(O.ROOT, "tests", "golden", "b200gen_spmv_csr.gen.cpp")).read()
    # the reference generator's ABI: infer_interface order, harnessgen kind types
    assert ('extern "C" void b200gen_spmv_csr(std::int64_t rows, double* output, const std::int64_t* row_ptr, '
            'const double* val, const double* x, const std::int64_t* col_ind)') in src


@pytest.mark.gpu
def test_generated_harness_parity_on_gpu():
    L = C.CDLL(GEN_LIB)
    f = L.b200gen_spmv_csr
    f.restype = None
    f.argtypes = [C.c_int64, O.f64p, O.i64p, O.f64p, O.f64p, O.i64p]
    for name, case in O.all_golden_cases()[:40]:
        c = O.case_arrays(case)
        y = np.full(c["rows"], np.nan)
        f(c["rows"], O.ptr(y), O.ptr(c["row_ptr"]), O.ptr(c["val"]), O.ptr(c["x"]), O.ptr(c["col_ind"]))
        bound = O.spmv_csr(c["row_ptr"], c["col_ind"], np.abs(c["val"]), np.abs(c["x"]))
        assert np.all(np.abs(y - c["y_csr"]) <= 1e-12 * bound), name
    rng = np.random.default_rng(4)
    n = 5000
    lens = rng.integers(0, 50, n)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = rng.integers(0, n, int(rp[-1])).astype(np.int64)
    val = rng.uniform(-1, 1, int(rp[-1]))
    x = np.zeros(n)
    for it in range(3):  # resident matrix, x rewritten each call (checksum strategy sees it)
        x[:] = rng.uniform(-1, 1, n)
        y = np.zeros(n)
        f(n, O.ptr(y), O.ptr(rp), O.ptr(val), O.ptr(x), O.ptr(ci))
        ref = O.spmv_csr(rp, ci, val, x)
        assert np.all(np.abs(y - ref) <= 1e-12 * O.spmv_csr(rp, ci, np.abs(val), np.abs(x)))
