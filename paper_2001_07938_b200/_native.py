"""ctypes binding of liblilac_b200.so (the C ABI in include/lilac_b200.h).

The native library is the product: there is no Python or CPU fallback. If it
is missing this module raises at import, naming the build command.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# LILAC_B200_LIB: an experiment build (tools/build_variant.py); default in-tree
LIB_PATH = os.environ.get("LILAC_B200_LIB") or os.path.join(PKG, "liblilac_b200.so")

i64 = C.c_int64
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


class RegionStats(C.Structure):
    _fields_ = [("region", C.c_char * 64), ("n_construct", i64), ("n_update", i64), ("n_destruct", i64),
                ("bytes_h2d", i64), ("bytes_d2h", i64), ("bytes_d2d", i64), ("strategy", C.c_int32), ("fell_back", C.c_int32),
                ("streaming", C.c_int32), ("constructed", C.c_int32)]


class HarnessStats(C.Structure):
    _fields_ = [("harness", C.c_char * 32), ("calls", i64), ("t_total_ms", C.c_double),
                ("t_poll_ms", C.c_double), ("t_kernel_ms", C.c_double), ("t_writeback_ms", C.c_double),
                ("bytes_h2d", i64), ("bytes_d2h", i64), ("bytes_d2d", i64)]


class B200Buf(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("bytes", C.c_size_t)]


class MatrixInfo(C.Structure):
    _fields_ = [("rows", i64), ("cols", i64), ("nnz", i64), ("max_row", i64), ("format", C.c_int32),
                ("col_bytes", C.c_int32), ("kernel", C.c_int32), ("lanes", C.c_int32),
                ("device_bytes", i64)]


# name -> (restype, argtypes); mirrors include/lilac_b200.h
SIGNATURES = {
    # 1. harness entry points
    "b200_spmv_csr": (None, [i64, f64p, i64p, f64p, f64p, i64p]),
    "b200_spmv_jds": (None, [i64, f64p, i64p, i64p, f64p, i64p, f64p, i64p]),
    "b200_dot": (None, [f64p, i64, f64p, f64p]),
    "b200_gemm": (None, [i64, i64, f64p, i64, f64p, f64p]),
    "b200_axpy": (None, [i64, f64p, C.c_double, f64p]),
    "b200_xpay": (None, [i64, f64p, C.c_double, f64p]),
    # 2. runtime control
    "b200_init": (C.c_int, [C.c_int]),
    "b200_shutdown": (None, []),
    "b200_set_error_mode": (None, [C.c_int]),
    "b200_last_error": (C.c_char_p, []),
    "b200_last_error_code": (C.c_char_p, []),
    "b200_set_kernel": (C.c_int, [C.c_char_p]),
    "b200_set_strategy": (C.c_int, [C.c_char_p]),
    "b200_set_exact_blas": (None, [C.c_int]),
    "b200_set_writeback": (C.c_int, [C.c_char_p]),
    "b200_set_profiling": (None, [C.c_int]),
    "b200_host_sync": (C.c_int, [vp, C.c_size_t]),
    "b200_host_forget": (C.c_int, [vp, C.c_size_t]),
    "b200_host_will_write": (C.c_int, [vp, C.c_size_t]),
    "b200_lazy_counters": (C.c_int, [C.POINTER(C.c_int64)] * 6),
    "b200_version": (C.c_char_p, []),
    # 3. counters
    "b200_region_stats_get": (C.c_int, [C.POINTER(RegionStats), C.c_int]),
    "b200_harness_stats_get": (C.c_int, [C.POINTER(HarnessStats), C.c_int]),
    "b200_stats_reset": (None, []),
    "b200_marshal_counters": (C.c_int, [i64p, i64p, i64p, i64p]),
    "b200_dma_visible_regions": (i64, []),
    "b200_host_profile": (C.c_int, [i64p, i64p, C.c_int]),
    # 4. resident device API
    "b200_matrix_create_csr": (C.c_int, [C.POINTER(vp), i64, i64p, i64p, f64p]),
    "b200_matrix_create_jds": (C.c_int, [C.POINTER(vp), i64, i64p, i64p, f64p, i64p, i64p]),
    "b200_matrix_free": (None, [vp]),
    "b200_matrix_info_get": (C.c_int, [vp, C.POINTER(MatrixInfo)]),
    "b200_spmv_device": (C.c_int, [vp, vp, vp, vp]),
    "b200_dot_device": (C.c_int, [vp, vp, i64, vp, vp]),
    "b200_gemm_device": (C.c_int, [i64, i64, i64, vp, vp, vp, C.c_int, vp]),
    "b200_axpy_device": (C.c_int, [i64, vp, C.c_double, vp, vp]),
    "b200_matrix_create_stencil27": (C.c_int, [C.POINTER(C.c_void_p), i64, C.c_double, C.c_double]),
    "b200_matrix_create_stencil27_rows": (C.c_int, [C.POINTER(C.c_void_p), i64, i64, i64, C.c_double, C.c_double]),
    "b200_pagerank_device": (C.c_int, [vp, C.c_double, C.c_int, vp, vp, vp]),
    "b200_pagerank_step_device": (C.c_int, [vp, C.c_double, vp, vp, vp]),
    "b200_cg_solve": (C.c_int, [vp, vp, C.c_int, vp, C.POINTER(C.c_double)]),
    "b200_dbuf_alloc": (C.c_int, [C.POINTER(B200Buf), C.c_size_t]),
    "b200_dbuf_upload": (C.c_int, [C.POINTER(B200Buf), vp, C.c_size_t]),
    "b200_dbuf_download": (C.c_int, [vp, C.POINTER(B200Buf), C.c_size_t]),
    "b200_dbuf_free": (None, [C.POINTER(B200Buf)]),
    "b200_spmv_csr_dev": (C.c_int, [i64, i64, i64, vp, vp, vp, vp, vp]),
    # 5. NPB CG driver
    "b200_cg_create": (C.c_int, [C.POINTER(vp), vp]),
    "b200_cg_free": (None, [vp]),
    "b200_cg_reset": (C.c_int, [vp, vp]),
    "b200_cg_outer": (C.c_int, [vp, C.c_int, C.c_double, vp]),
    "b200_cg_step": (C.c_int, [vp, vp]),
    "b200_cg_result": (C.c_int, [vp, f64p, f64p]),
    "b200_cg_start": (C.c_int, [vp, vp, vp]),
    "b200_cg_finish": (C.c_int, [vp, vp]),
    "b200_cg_scalars": (C.c_int, [vp, vp, f64p, f64p]),
    "b200_npb_cg": (C.c_int, [vp, C.c_int, C.c_double, f64p, f64p]),
    # 6. workloads
    "b200_gen_npb": (C.c_int, [i64, C.c_int, C.c_double, i64p, i64p, f64p, i64p]),
    "b200_gen_kronecker": (C.c_int, [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_double, i64p, i64p,
                                     f64p]),
    # 7. sharding
    "b200_partition_rows": (None, [i64, i64p, C.c_int, i64p]),
    "b200_shard_footprint": (None, [i64, i64p, i64p, i64p, i64p]),
    "b200_dist_send_ranges": (None, [C.c_int, i64p, i64p, i64p, i64p]),
    "b200_dist_nccl_id": (C.c_int, [vp]),
    "b200_dist_cg_create_nccl": (C.c_int, [C.POINTER(vp), C.c_int, C.c_int, vp, i64, i64p, i64p, i64p, f64p]),
    "b200_dist_cg_create_local": (C.c_int, [C.POINTER(vp), C.c_int, i64, i64p, i64p, f64p]),
    "b200_dist_cg_free": (None, [vp]),
    "b200_dist_cg_create_stencil27_nccl": (C.c_int, [C.POINTER(vp), C.c_int, C.c_int, vp, i64, C.c_double,
                                                     C.c_double]),
    "b200_dist_cg_create_stencil27_local": (C.c_int, [C.POINTER(vp), C.c_int, i64, C.c_double, C.c_double]),
    "b200_dist_cg_bounds": (C.c_int, [vp, i64p]),
    "b200_dist_cg_start_rowsum": (C.c_int, [vp, vp]),
    "b200_dist_cg_start": (C.c_int, [vp, vp]),
    "b200_dist_cg_step": (C.c_int, [vp, vp]),
    "b200_dist_cg_finish": (C.c_int, [vp, vp]),
    "b200_dist_cg_scalars": (C.c_int, [vp, vp, f64p, f64p]),
    "b200_dist_cg_reset": (C.c_int, [vp, vp]),
    "b200_dist_cg_outer": (C.c_int, [vp, C.c_int, C.c_double, vp]),
    "b200_dist_cg_result": (C.c_int, [vp, f64p, f64p]),
    "b200_dist_cg_load_x": (C.c_int, [vp, vp, vp]),
    "b200_dist_cg_use_p2p_local": (C.c_int, [vp]),
    "b200_dist_cg_p2p_export": (C.c_int, [vp, vp]),
    "b200_dist_cg_p2p_attach": (C.c_int, [vp, vp]),
    "b200_dist_cg_transport": (C.c_int, [vp]),
    "b200_dist_cg_set_fused": (C.c_int, [vp, C.c_int]),
    "b200_dist_cg_fused": (C.c_int, [vp]),
    "b200_dist_npb": (C.c_int, [vp, C.c_int, C.c_double, f64p, f64p]),
    "b200_dist_cg_info": (C.c_int, [vp, C.c_int, i64p, i64p, i64p, C.POINTER(C.c_int32)]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is not built; run `python -m paper_2001_07938_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def ptr(a):
    """ctypes pointer to a numpy array's data (int64 / float64), or None."""
    if a is None:
        return None
    import numpy as np
    if a.dtype == np.int64:
        return a.ctypes.data_as(i64p)
    if a.dtype == np.float64:
        return a.ctypes.data_as(f64p)
    raise TypeError(f"unsupported dtype {a.dtype}")


class B200Error(RuntimeError):
    def __init__(self, code: str, message: str):
        super().__init__(f"{code}: {message}")
        self.code = code


def check(rc: int = 0):
    """Raise B200Error if the last C-ABI call failed (error mode RETURN)."""
    L = lib()
    code = L.b200_last_error_code().decode()
    if rc != 0 or code:
        raise B200Error(code or "Error", L.b200_last_error().decode())
