"""Randomised stress of the C-ABI harnesses on the B200: interleaved CSR / JDS
/ dot / axpy / xpay / gemm calls on arrays that are reused, rewritten by the
host, freed and reallocated (malloc'd numpy and page-aligned mmap arrays),
with lazy and eager write-back toggled. Every result is checked against the
oracle; the marshal runtime's guards, mirrors and lazy ranges must never serve
stale bytes or fault on recycled memory."""
import gc

import numpy as np
import pytest

import oracle_lib as O
from paper_2001_07938_b200 import _native as N
from paper_2001_07938_b200 import harness as H

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _errors_return():
    H.set_errors_return(True)
    N.lib().b200_set_kernel(b"auto")
    N.lib().b200_set_exact_blas(0)
    yield
    H.host_sync()
    H.host_forget()
    H.set_writeback("eager")


def rand_csr(rng, rows, cols, mean):
    lens = rng.integers(0, 2 * mean + 1, rows)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = rng.integers(0, cols, int(rp[-1])).astype(np.int64)
    val = rng.uniform(-1, 1, int(rp[-1]))
    return rp, ci, val


def close(a, b, scale):
    return np.all(np.abs(a - b) <= 1e-12 * scale + 1e-300)


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_interleaved_harness_calls_stay_coherent(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20_000, 60_000))
    rp, ci, val = rand_csr(rng, n, n, 6)
    perm, nzcnt, jd_ptr, jval, jcol = O.jds_from_csr(rp, ci, val)
    abs_val = np.abs(val)

    def alloc(k):
        return H.page_aligned(k) if rng.random() < 0.5 else np.zeros(k)

    vecs = [alloc(n) for _ in range(4)]
    for v in vecs:
        v[:] = rng.uniform(-1, 1, n)
    for step in range(250):
        if rng.random() < 0.1:
            H.set_writeback("lazy" if rng.random() < 0.5 else "eager")
        op = rng.integers(0, 7)
        i, j = rng.choice(4, 2, replace=False)
        x, y = vecs[i], vecs[j]
        if op == 0:  # CSR SpMV y = A x
            xs = np.array(x)
            H.spmv_csr(n, y, rp, val, x, ci)
            ref = O.spmv_csr(rp, ci, val, xs)
            assert close(y, ref, O.spmv_csr(rp, ci, abs_val, np.abs(xs))), (step, op)
        elif op == 1:  # JDS SpMV (bit-exact)
            xs = np.array(x)
            H.spmv_jds(n, y, nzcnt, perm, jval, jd_ptr, x, jcol)
            assert O.same_bits(np.array(y), O.spmv_csr(rp, ci, val, xs)) or close(
                y, O.spmv_csr(rp, ci, val, xs), O.spmv_csr(rp, ci, abs_val, np.abs(xs))), (step, op)
        elif op == 2:  # dot
            r = H.dotproduct(n, x, y)
            assert abs(r - O.dot(np.array(x), np.array(y))) <= 1e-12 * float(np.abs(np.array(x) * np.array(y)).sum())
        elif op == 3:  # axpy y += a x (bit-exact)
            a = float(rng.uniform(-1, 1))
            ref = O.axpy(np.array(y), a, np.array(x))  # returns y + a*x (a copy)
            H.axpy(n, y, a, x)
            assert O.same_bits(np.array(y), ref), (step, op)
        elif op == 4:  # xpay y = x + b y (bit-exact)
            b = float(rng.uniform(-1, 1))
            ref = np.array(x) + b * np.array(y)
            H.xpay(n, y, b, x)
            assert O.same_bits(np.array(y), ref), (step, op)
        elif op == 5:  # host rewrites part of an array
            lo = int(rng.integers(0, n))
            y[lo:lo + int(rng.integers(1, 5000))] = rng.uniform(-1, 1)
        else:  # free and reallocate (stale guards / mirrors / lazy ranges)
            H.host_sync(y)
            H.host_forget(y)
            vecs[j] = alloc(n)
            vecs[j][:] = rng.uniform(-1, 1, n)
            gc.collect()
    H.host_sync()


def test_gemm_between_vector_calls():
    rng = np.random.default_rng(7)
    for k in range(6):
        nn, mm, pp = (int(v) for v in rng.integers(1, 200, 3))
        a = rng.uniform(-1, 1, nn * pp)
        b = rng.uniform(-1, 1, pp * mm)
        c = np.zeros(nn * mm)
        H.gemm(nn, mm, c, pp, a, b)
        ref = O.gemm(nn, mm, pp, a, b)
        assert close(c, ref, O.gemm(nn, mm, pp, np.abs(a), np.abs(b)))
        d = H.dotproduct(nn * mm, c, c)
        assert abs(d - O.dot(ref, ref)) <= 1e-11 * O.dot(np.abs(ref), np.abs(ref))
