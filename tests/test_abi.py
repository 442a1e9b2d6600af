"""CPU-side checks of the C ABI library (no GPU calls).

* liblilac_b200.so loads and exports every function include/lilac_b200.h declares;
* host-side index work (row partition, NPB makea) is bit-exact against the oracle;
* with no GPU, harness calls fail loudly (DeviceError) — never a CPU fallback.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle_lib as O
from paper_2001_07938_b200 import _native as N
from paper_2001_07938_b200 import device as D
from paper_2001_07938_b200 import harness as H

HEADER = os.path.join(O.ROOT, "include", "lilac_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(b200_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = N.lib()
    names = declared_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and the Python binding covers the same set
    assert set(names) == set(N.SIGNATURES), set(names) ^ set(N.SIGNATURES)


def test_version_string():
    assert N.lib().b200_version().decode().startswith("lilac-b200")


def test_harness_signatures_match_reference_infer_interface():
    """The entry points take their parameters in the reference's
    infer_interface order (tests/golden/abi.json, written by the reference)."""
    sigs = O.golden("abi.json")["signatures"]
    kinds = {"scalar-int": N.i64, "array-int": N.i64p, "array-float-in": N.f64p, "array-float-out": N.f64p}
    table = {"spmv_csr": "b200_spmv_csr", "spmv_jds": "b200_spmv_jds", "dotproduct": "b200_dot", "gemm": "b200_gemm"}
    for comp, fn in table.items():
        want = [kinds[k] for _, k in sigs[comp]]
        got = N.SIGNATURES[fn][1]
        assert got == want, (comp, got, want)
    # the header spells the same parameter names in the same order
    text = open(HEADER).read()
    for comp, fn in table.items():
        m = re.search(fn + r"\(([^)]*)\)", text)
        params = [p.strip().split()[-1].lstrip("*") for p in m.group(1).split(",")]
        assert params == [n for n, _ in sigs[comp]], (fn, params)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 7, 8])
def test_partition_rows_bit_exact_vs_oracle(k):
    rng = np.random.default_rng(k)
    for rows in (0, 1, 5, 1000):
        lens = rng.integers(0, 60, size=rows)
        lens[rng.random(rows) < 0.1] = 0
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        assert np.array_equal(D.partition_rows(rp, k), O.partition_rows(rp, k))


@pytest.mark.parametrize("cls", ["S", "A", "C"])
def test_gen_npb_bit_exact_vs_oracle_makea(cls):
    na, nonzer, _, shift, _ = D.NPB_CLASSES[cls]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    orp, oci, oval = O.npb_makea(na, nonzer, shift)
    assert np.array_equal(rp, orp)
    assert np.array_equal(ci, oci)
    assert O.same_bits(val, oval)


def test_harness_registry_mirror():
    reg = H.register_b200_harnesses(H.HarnessRegistry())
    assert reg.names() == ["lilac.dotproduct", "lilac.gemm", "lilac.spmv_csr", "lilac.spmv_jds"]
    with pytest.raises(KeyError):
        reg.add("lilac.spmv_csr", lambda: None)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    H.set_errors_return(True)
    try:
        y = np.zeros(5)
        rp = np.array([0, 2, 4, 7, 8, 10], np.int64)
        ci = np.array([0, 2, 1, 3, 1, 2, 3, 3, 2, 4], np.int64)
        val = np.ones(10)
        with pytest.raises(H.B200Error) as e:
            H.spmv_csr(5, y, rp, val, np.ones(5), ci)
        assert e.value.code == "DeviceError"
        assert np.all(y == 0)  # outputs untouched
    finally:
        H.set_errors_return(False)


def test_python_binding_checks_arguments_before_calling():
    """The CPython binding (csrc/pyext/harness_module.c) is built and rejects
    wrong dtypes / layouts / read-only outputs without calling the library."""
    import numpy as np
    from paper_2001_07938_b200 import harness as H
    E = H._ext()
    assert E is not None, "paper_2001_07938_b200/_harness*.so not built"
    rp = np.array([0, 1], np.int64)
    ci = np.array([0], np.int64)
    val = np.ones(1)
    x = np.ones(1)
    with pytest.raises(TypeError, match="output"):
        H.spmv_csr(1, np.zeros(1, np.float32), rp, val, x, ci)
    with pytest.raises(TypeError, match="row_ptr"):
        H.spmv_csr(1, np.zeros(1), rp.astype(np.int32), val, x, ci)
    with pytest.raises(TypeError, match="x"):
        H.spmv_csr(1, np.zeros(1), rp, val, np.ones(4)[::2], ci)
    ro = np.zeros(1)
    ro.flags.writeable = False
    with pytest.raises(TypeError, match="output"):
        H.spmv_csr(1, ro, rp, val, x, ci)
    with pytest.raises(TypeError, match="y"):
        H.axpy(1, ro, 1.0, x)


def test_harness_tracks_array_lifetimes():
    """Every array handed to a harness binding gets a finalizer on its owner
    that forgets the range (guards, lazy pages, device copy) when it dies, so
    protected pages never outlive the memory (harness.py _track)."""
    import gc

    import numpy as np

    from paper_2001_07938_b200 import harness as H
    base = np.arange(4096, dtype=np.float64)
    view = base[8:1000]
    H._track(view, view[3:5], np.zeros(0))
    assert id(base) in H._TRACKED and len([k for k in H._TRACKED if k == id(base)]) == 1
    k = id(base)
    del base, view
    gc.collect()
    assert k not in H._TRACKED
