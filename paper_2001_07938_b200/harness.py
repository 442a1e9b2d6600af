"""Host-side mirror of the reference's harness interface for the B200 path.

The reference exposes this path as named callables: the interpreter's
``HarnessRegistry`` holds ``"lilac.<computation>"`` entries whose arguments
arrive in ``infer_interface`` order (src/interp.cpp:330-389,
include/lilac/interp.hpp:73-83), and compiled programs call the generated
``extern "C"`` harness symbols (src/harnessgen.cpp:86-92). This module offers
the same names, argument order and error behaviour over numpy arrays, backed
by liblilac_b200.so: every call goes through the C ABI (no CPU path).

    spmv_csr(rows, output, row_ptr, val, x, col_ind)
    spmv_jds(rows, output, nzcnt, perm, val, jd_ptr, x, col_ind)
    dotproduct(length, a, b) -> float        (scalar-result protocol: the
                                             result slot is synthesized,
                                             interp.cpp:335-346, 385)
"""
from __future__ import annotations

import weakref

import numpy as np

from . import _native as N

__all__ = ["spmv_csr", "spmv_jds", "dotproduct", "gemm", "axpy", "xpay", "HarnessRegistry",
           "register_b200_harnesses", "region_stats", "harness_stats", "B200Error", "set_errors_return",
           "set_writeback", "host_sync", "host_forget", "lazy_counters", "page_aligned"]

B200Error = N.B200Error


def _f64(a, name, writable=False):
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
        raise TypeError(f"{name}: expected a C-contiguous float64 numpy array")
    if writable and not a.flags.writeable:
        raise TypeError(f"{name}: output must be writable")
    return a


def _i64(a, name):
    if not isinstance(a, np.ndarray) or a.dtype != np.int64 or not a.flags.c_contiguous:
        raise TypeError(f"{name}: expected a C-contiguous int64 numpy array")
    return a


def set_errors_return(on: bool = True):
    """Return-with-exception instead of abort on harness errors (tests)."""
    N.lib().b200_set_error_mode(1 if on else 0)


def _ext():
    """The CPython binding (csrc/pyext/harness_module.c) — same C-ABI calls
    without ctypes' per-argument marshalling cost; None if not built."""
    global _EXT
    if _EXT is False:
        try:
            N.lib()  # loads liblilac_b200.so (and fails loudly if it is missing)
            from . import _harness as E
            E.set_error_class(B200Error)
            _EXT = E
        except ImportError:
            _EXT = None
    return _EXT


_EXT = False


# ---- host memory lifetime ----------------------------------------------------------
# The marshaling runtime write-protects pages of the arrays it caches (change
# detection) and, in lazy mode, leaves output pages inaccessible until read.
# A C caller owns its arrays for as long as it uses the harness; a numpy array
# can die and its memory be reused by the allocator while the pages are still
# protected — a later write by the kernel into that memory (a read() into a
# buffer) then fails with EFAULT instead of faulting into the handler. So the
# first time an array's memory reaches the harness, a finalizer on its owner
# forgets the range (guards dropped, pages restored, cached device copy
# released) when the owner dies.
_TRACKED: dict = {}


def _owner(a):
    o = a
    while isinstance(o, np.ndarray) and o.base is not None:
        o = o.base
    return o


def _track(*arrays):
    for a in arrays:
        if not isinstance(a, np.ndarray) or a.nbytes == 0:
            continue
        o = _owner(a)
        k = id(o)
        if k in _TRACKED:
            continue
        try:
            if isinstance(o, np.ndarray):
                addr, size = o.ctypes.data, o.nbytes
            else:  # a buffer object (mmap, bytearray, ...): its whole range
                whole = np.frombuffer(o, np.uint8)
                addr, size = whole.ctypes.data, whole.nbytes
            _TRACKED[k] = weakref.finalize(o, _untrack, k, addr, size)
        except (TypeError, ValueError):
            pass  # not weak-referenceable: nothing to hook


def _untrack(k, addr, size):
    _TRACKED.pop(k, None)
    _forget_addr(addr, size)


def spmv_csr(rows, output, row_ptr, val, x, col_ind):
    _track(output, row_ptr, val, x, col_ind)
    E = _ext()
    if E is not None:
        return E.spmv_csr(int(rows), output, row_ptr, val, x, col_ind)
    L = N.lib()
    L.b200_spmv_csr(int(rows), N.ptr(_f64(output, "output", True)), N.ptr(_i64(row_ptr, "row_ptr")),
                    N.ptr(_f64(val, "val")), N.ptr(_f64(x, "x")), N.ptr(_i64(col_ind, "col_ind")))
    N.check()


def spmv_jds(rows, output, nzcnt, perm, val, jd_ptr, x, col_ind):
    _track(output, nzcnt, perm, val, jd_ptr, x, col_ind)
    E = _ext()
    if E is not None:
        return E.spmv_jds(int(rows), output, nzcnt, perm, val, jd_ptr, x, col_ind)
    L = N.lib()
    L.b200_spmv_jds(int(rows), N.ptr(_f64(output, "output", True)), N.ptr(_i64(nzcnt, "nzcnt")),
                    N.ptr(_i64(perm, "perm")), N.ptr(_f64(val, "val")), N.ptr(_i64(jd_ptr, "jd_ptr")),
                    N.ptr(_f64(x, "x")), N.ptr(_i64(col_ind, "col_ind")))
    N.check()


def dotproduct(length, a, b) -> float:
    _track(a, b)
    E = _ext()
    if E is not None:
        return E.dotproduct(int(length), a, b)
    res = np.zeros(1, np.float64)
    N.lib().b200_dot(N.ptr(res), int(length), N.ptr(_f64(a, "a")), N.ptr(_f64(b, "b")))
    N.check()
    return float(res[0])


def gemm(n, m, c, p, a, b):
    """c[i*m + j] = sum_k a[i*p + k] * b[k*m + j] (kernels.lilac:14-19)."""
    _track(c, a, b)
    E = _ext()
    if E is not None:
        return E.gemm(int(n), int(m), c, int(p), a, b)
    for arr, need, name in ((c, n * m, "c"), (a, n * p, "a"), (b, p * m, "b")):
        if _f64(arr, name, name == "c").size < need:
            raise ValueError("gemm: arrays shorter than n*m (c), n*p (a), p*m (b)")
    N.lib().b200_gemm(int(n), int(m), N.ptr(c), int(p), N.ptr(a), N.ptr(b))
    N.check()


def axpy(n, y, alpha, x):
    _track(y, x)
    E = _ext()
    if E is not None:
        return E.axpy(int(n), y, float(alpha), x)
    N.lib().b200_axpy(int(n), N.ptr(_f64(y, "y", True)), float(alpha), N.ptr(_f64(x, "x")))
    N.check()


def xpay(n, y, beta, x):
    _track(y, x)
    E = _ext()
    if E is not None:
        return E.xpay(int(n), y, float(beta), x)
    N.lib().b200_xpay(int(n), N.ptr(_f64(y, "y", True)), float(beta), N.ptr(_f64(x, "x")))
    N.check()


def set_writeback(mode: str):
    """"eager" (the reference's behaviour) or "lazy" (outputs stay on the
    device until the host touches them; include/lilac_b200.h)."""
    N.check(N.lib().b200_set_writeback(mode.encode()))


def host_sync(a=None):
    """Materialise lazy write-back bytes of `a` (all when None) — needed before
    handing the array to DMA or a system call."""
    if a is None:
        N.check(N.lib().b200_host_sync(None, 0))
    else:
        N.check(N.lib().b200_host_sync(N.ptr(a), a.nbytes))


def host_will_write(a):
    """`a` is about to be written by something that does not fault (a system
    call such as os.readv / file.readinto, or DMA): fill its lazy bytes, lift
    the change-detection guards (a guarded page makes the system call fail
    with EFAULT) and mark it changed (include/lilac_b200.h)."""
    N.check(N.lib().b200_host_will_write(N.ptr(a), a.nbytes))


def host_forget(a=None):
    """Drop every binding / mirror / guard / lazy range over `a` (all when
    None) before its memory is freed or recycled (include/lilac_b200.h)."""
    if a is None:
        N.check(N.lib().b200_host_forget(None, 0))
    else:
        N.check(N.lib().b200_host_forget(N.ptr(a), a.nbytes))


def lazy_counters():
    import ctypes as C
    v = [C.c_int64() for _ in range(6)]
    N.lib().b200_lazy_counters(*[C.byref(x) for x in v])
    keys = ["ranges", "fault_fills", "explicit_fills", "cancelled", "bytes_deferred", "bytes_filled"]
    return {k: x.value for k, x in zip(keys, v)}


def page_aligned(n, dtype=np.float64):
    """A zeroed array whose data starts on a page boundary (lazy write-back
    defers every whole page of an output; on an unaligned array the two
    partial edge pages are written at once)."""
    import mmap
    dt = np.dtype(dtype)
    nbytes = max(int(n) * dt.itemsize, 1)
    size = (nbytes + mmap.PAGESIZE - 1) // mmap.PAGESIZE * mmap.PAGESIZE
    buf = mmap.mmap(-1, size)
    a = np.frombuffer(buf, dtype=dt, count=int(n))
    # unmapped when the last view dies: forget it first (no stale guard or
    # lazy fill may outlive the mapping)
    addr = a.ctypes.data
    weakref.finalize(buf, _forget_addr, addr, size)
    return a


def _forget_addr(addr, size):
    try:
        N.lib().b200_host_forget(addr, size)
    except Exception:  # interpreter teardown
        pass


class HarnessRegistry:
    """Name -> callable table (reference interp.hpp:75-83: add/find/names;
    add() of an existing name raises, like DuplicateRegistration)."""

    def __init__(self):
        self._fns = {}

    def add(self, name, fn):
        if name in self._fns:
            raise KeyError(f"DuplicateRegistration: harness '{name}' already registered")
        self._fns[name] = fn

    def find(self, name):
        return self._fns.get(name)

    def names(self):
        return sorted(self._fns)


def register_b200_harnesses(reg: HarnessRegistry, computations=("spmv_csr", "spmv_jds", "dotproduct", "gemm")):
    """Counterpart of interp::register_reference_harnesses (interp.cpp:330):
    registers the B200 harnesses under "lilac.<computation>"."""
    table = {"spmv_csr": spmv_csr, "spmv_jds": spmv_jds, "dotproduct": dotproduct, "gemm": gemm}
    for c in computations:
        reg.add("lilac." + c, table[c])
    return reg


def region_stats():
    """Marshal counters per region: the `run --stats` rows of the reference CLI
    (tools/lilac_main.cpp:599-612) plus transfer bytes."""
    L = N.lib()
    n = L.b200_region_stats_get(None, 0)
    arr = (N.RegionStats * max(n, 1))()
    L.b200_region_stats_get(arr, n)
    names = ["pageprotect", "checksum", "exact", "naive", "hybrid"]
    return {r.region.decode(): {"n_construct": r.n_construct, "n_update": r.n_update, "n_destruct": r.n_destruct,
                                "bytes_h2d": r.bytes_h2d, "bytes_d2h": r.bytes_d2h, "bytes_d2d": r.bytes_d2d,
                                "strategy": names[r.strategy], "fell_back": bool(r.fell_back),
                                "streaming": bool(r.streaming), "constructed": bool(r.constructed)}
            for r in arr[:n]}


def harness_stats():
    L = N.lib()
    n = L.b200_harness_stats_get(None, 0)
    arr = (N.HarnessStats * max(n, 1))()
    L.b200_harness_stats_get(arr, n)
    return {h.harness.decode(): {"calls": h.calls, "t_total_ms": h.t_total_ms, "t_poll_ms": h.t_poll_ms,
                                 "t_kernel_ms": h.t_kernel_ms, "t_writeback_ms": h.t_writeback_ms,
                                 "bytes_h2d": h.bytes_h2d, "bytes_d2h": h.bytes_d2h, "bytes_d2d": h.bytes_d2d}
            for h in arr[:n]}
