"""Resident-device API (section 4-7 of include/lilac_b200.h) for drivers,
benchmarks and tests. Device pointers / streams are plain integers (e.g.
``torch.Tensor.data_ptr()`` and ``torch.cuda.Stream.cuda_stream``)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


class Matrix:
    """A CSR or JDS matrix uploaded once and kept resident in HBM."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def csr(cls, row_ptr, col_ind, val, rows=None):
        rows = len(row_ptr) - 1 if rows is None else rows
        h = C.c_void_p()
        rc = N.lib().b200_matrix_create_csr(C.byref(h), rows, N.ptr(row_ptr), N.ptr(col_ind), N.ptr(val))
        N.check(rc)
        return cls(h)

    @classmethod
    def jds(cls, nzcnt, perm, val, jd_ptr, col_ind):
        h = C.c_void_p()
        rc = N.lib().b200_matrix_create_jds(C.byref(h), len(perm), N.ptr(nzcnt), N.ptr(perm), N.ptr(val),
                                            N.ptr(jd_ptr), N.ptr(col_ind))
        N.check(rc)
        return cls(h)

    @classmethod
    def stencil27(cls, nx: int, diag: float = 26.1, offdiag: float = -1.0):
        """The 27-point stencil operator on an nx^3 grid, generated in HBM."""
        h = C.c_void_p()
        N.check(N.lib().b200_matrix_create_stencil27(C.byref(h), int(nx), float(diag), float(offdiag)))
        return cls(h)

    @classmethod
    def stencil27_rows(cls, nx: int, r0: int, r1: int, diag: float = 26.1, offdiag: float = -1.0):
        """Rows [r0, r1) of `stencil27(nx)` (all nx^3 columns): one row shard."""
        h = C.c_void_p()
        N.check(N.lib().b200_matrix_create_stencil27_rows(C.byref(h), int(nx), int(r0), int(r1), float(diag),
                                                          float(offdiag)))
        return cls(h)

    @property
    def handle(self):
        return self._h

    def pagerank(self, damping: float, iters: int, x_ptr: int, work_ptr: int, stream: int = 0):
        """`iters` steps of x = damping*(A x) + (1-damping)/n on device vectors."""
        N.check(N.lib().b200_pagerank_device(self._h, float(damping), int(iters), C.c_void_p(x_ptr),
                                             C.c_void_p(work_ptr), C.c_void_p(stream)))

    def pagerank_step(self, damping: float, x_ptr: int, y_ptr: int, stream: int = 0):
        """y = damping*(A x) + (1-damping)/n into another device vector."""
        N.check(N.lib().b200_pagerank_step_device(self._h, float(damping), C.c_void_p(x_ptr), C.c_void_p(y_ptr),
                                                  C.c_void_p(stream)))

    def info(self) -> dict:
        i = N.MatrixInfo()
        N.check(N.lib().b200_matrix_info_get(self._h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in N.MatrixInfo._fields_}

    def spmv(self, x_ptr: int, y_ptr: int, stream: int = 0):
        rc = N.lib().b200_spmv_device(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), C.c_void_p(stream))
        if rc:
            N.check(rc)

    def free(self):
        if self._h:
            N.lib().b200_matrix_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def dot(a_ptr: int, b_ptr: int, n: int, out_ptr: int, stream: int = 0):
    N.check(N.lib().b200_dot_device(C.c_void_p(a_ptr), C.c_void_p(b_ptr), n, C.c_void_p(out_ptr),
                                    C.c_void_p(stream)))


def gemm(n: int, m: int, p: int, a_ptr: int, b_ptr: int, c_ptr: int, exact: bool = False, stream: int = 0):
    """c = a b on device buffers (row-major n x p times p x m)."""
    N.check(N.lib().b200_gemm_device(n, m, p, C.c_void_p(a_ptr), C.c_void_p(b_ptr), C.c_void_p(c_ptr),
                                     1 if exact else 0, C.c_void_p(stream)))


class CG:
    """NPB CG solver state over a resident CSR matrix."""

    def __init__(self, A: Matrix):
        h = C.c_void_p()
        N.check(N.lib().b200_cg_create(C.byref(h), A.handle))
        self._h = h
        self.A = A

    def reset(self, stream: int = 0):
        N.check(N.lib().b200_cg_reset(self._h, C.c_void_p(stream)))

    def outer(self, shift: float, cgitmax: int = 25, stream: int = 0):
        rc = N.lib().b200_cg_outer(self._h, cgitmax, shift, C.c_void_p(stream))
        if rc:
            N.check(rc)

    def step(self, stream: int = 0):
        N.check(N.lib().b200_cg_step(self._h, C.c_void_p(stream)))

    def result(self):
        z = C.c_double()
        r = C.c_double()
        N.check(N.lib().b200_cg_result(self._h, C.byref(z), C.byref(r)))
        return z.value, r.value

    def start(self, b_ptr: int = 0, stream: int = 0):
        """x = b (device array; 0 keeps x), z = 0, r = p = b, rho = r.r."""
        N.check(N.lib().b200_cg_start(self._h, C.c_void_p(b_ptr or None), C.c_void_p(stream)))

    def finish(self, stream: int = 0):
        """rnorm = |b - A z| (read it with scalars())."""
        N.check(N.lib().b200_cg_finish(self._h, C.c_void_p(stream)))

    def scalars(self, stream: int = 0):
        """(rho, rnorm) on the host; synchronises `stream`."""
        rho, rn = C.c_double(), C.c_double()
        N.check(N.lib().b200_cg_scalars(self._h, C.c_void_p(stream), C.byref(rho), C.byref(rn)))
        return rho.value, rn.value

    def solve(self, b_ptr: int, iters: int, z_ptr: int = 0) -> float:
        """Plain CG on A z = b from z = 0 for `iters` steps; returns |b - A z|."""
        r = C.c_double()
        N.check(N.lib().b200_cg_solve(self._h, C.c_void_p(b_ptr), int(iters), C.c_void_p(z_ptr or None),
                                      C.byref(r)))
        return r.value

    def npb(self, niter: int, shift: float):
        z = C.c_double()
        r = C.c_double()
        N.check(N.lib().b200_npb_cg(self._h, niter, shift, C.byref(z), C.byref(r)))
        return z.value, r.value

    def free(self):
        if self._h:
            N.lib().b200_cg_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# NPB CG classes (NPB 3.x): na, nonzer, niter, shift, zeta_verify
NPB_CLASSES = {
    "S": (1400, 7, 15, 10.0, 8.5971775078648),
    "W": (7000, 8, 15, 12.0, 10.362595087124),
    "A": (14000, 11, 15, 20.0, 17.130235054029),
    "B": (75000, 13, 75, 60.0, 22.712745482631),
    "C": (150000, 15, 75, 110.0, 28.973605592845),
}


def gen_npb(na: int, nonzer: int, shift: float):
    """NPB makea via the native generator: (row_ptr, col_ind, val)."""
    L = N.lib()
    rp = np.zeros(na + 1, np.int64)
    nnz = np.zeros(1, np.int64)
    N.check(L.b200_gen_npb(na, nonzer, shift, N.ptr(rp), None, None, N.ptr(nnz)))
    ci = np.empty(int(nnz[0]), np.int64)
    val = np.empty(int(nnz[0]), np.float64)
    N.check(L.b200_gen_npb(na, nonzer, shift, N.ptr(rp), N.ptr(ci), N.ptr(val), N.ptr(nnz)))
    return rp, ci, val


def partition_rows(row_ptr, k: int):
    b = np.zeros(k + 1, np.int64)
    N.lib().b200_partition_rows(len(row_ptr) - 1, N.ptr(row_ptr), k, N.ptr(b))
    return b


class DistCG:
    """Row-sharded NPB CG (include/lilac_b200.h section 7).

    ``DistCG.local(k, row_ptr, col_ind, val)``: k shards on this GPU (device-copy
    exchange) — the sharded algorithm on one B200.
    ``DistCG.nccl(rank, world, nccl_id, n, bounds, row_ptr, col_ind, val)``: one
    shard per process; ``row_ptr`` covers this rank's rows only."""

    def __init__(self, handle, world):
        self._h = handle
        self.world = world

    @classmethod
    def local(cls, k, row_ptr, col_ind, val):
        h = C.c_void_p()
        N.check(N.lib().b200_dist_cg_create_local(C.byref(h), k, len(row_ptr) - 1, N.ptr(row_ptr),
                                                  N.ptr(col_ind), N.ptr(val)))
        return cls(h, k)

    @classmethod
    def nccl(cls, rank, world, nccl_id: bytes, n, bounds, row_ptr, col_ind, val):
        h = C.c_void_p()
        idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        N.check(N.lib().b200_dist_cg_create_nccl(C.byref(h), rank, world, idbuf, n, N.ptr(bounds),
                                                 N.ptr(row_ptr), N.ptr(col_ind), N.ptr(val)))
        return cls(h, world)

    @classmethod
    def stencil27_nccl(cls, rank, world, nccl_id: bytes, nx, diag=26.1, offdiag=-1.0):
        h = C.c_void_p()
        idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        N.check(N.lib().b200_dist_cg_create_stencil27_nccl(C.byref(h), rank, world, idbuf, nx, diag, offdiag))
        return cls(h, world)

    @classmethod
    def stencil27_local(cls, k, nx, diag=26.1, offdiag=-1.0):
        h = C.c_void_p()
        N.check(N.lib().b200_dist_cg_create_stencil27_local(C.byref(h), k, nx, diag, offdiag))
        return cls(h, k)

    @staticmethod
    def nccl_id() -> bytes:
        buf = C.create_string_buffer(128)
        N.check(N.lib().b200_dist_nccl_id(buf))
        return buf.raw

    def reset(self, stream: int = 0):
        N.check(N.lib().b200_dist_cg_reset(self._h, C.c_void_p(stream)))

    def outer(self, shift: float, cgitmax: int = 25, stream: int = 0):
        rc = N.lib().b200_dist_cg_outer(self._h, cgitmax, shift, C.c_void_p(stream))
        if rc:
            N.check(rc)

    def result(self):
        z, r = C.c_double(), C.c_double()
        N.check(N.lib().b200_dist_cg_result(self._h, C.byref(z), C.byref(r)))
        return z.value, r.value

    def use_p2p_local(self):
        """Exchange between the local shards through peer memory (p2p.cu)."""
        N.check(N.lib().b200_dist_cg_use_p2p_local(self._h))

    def p2p_export(self) -> bytes:
        """This rank's record for p2p_attach (208 bytes: three CUDA IPC
        handles and its column footprint)."""
        buf = C.create_string_buffer(208)
        N.check(N.lib().b200_dist_cg_p2p_export(self._h, buf))
        return buf.raw

    def p2p_attach(self, handles: bytes):
        """All ranks' records, rank-major (world x 208 bytes)."""
        N.check(N.lib().b200_dist_cg_p2p_attach(self._h, C.create_string_buffer(bytes(handles), len(handles))))

    def set_fused(self, on: bool):
        """The persistent sharded CG kernel (peer memory + tiled shards) on / off."""
        N.check(N.lib().b200_dist_cg_set_fused(self._h, 1 if on else 0))

    @property
    def fused(self) -> bool:
        """The last outer iteration ran the persistent sharded CG kernel."""
        return N.lib().b200_dist_cg_fused(self._h) == 1

    @property
    def transport(self) -> str:
        return {0: "local", 1: "nccl", 2: "p2p"}.get(N.lib().b200_dist_cg_transport(self._h), "?")

    def load_x(self, x_host_ptr: int, stream: int = 0):
        """x of this process's shards from host memory (its owned rows)."""
        N.check(N.lib().b200_dist_cg_load_x(self._h, C.c_void_p(x_host_ptr), C.c_void_p(stream)))

    def start_rowsum(self, stream: int = 0):
        """x = b = A 1, z = 0, r = p = b (plain CG, the stencil config)."""
        N.check(N.lib().b200_dist_cg_start_rowsum(self._h, C.c_void_p(stream)))

    def start(self, stream: int = 0):
        """b = the shards' x (load_x first), z = 0, r = p = b."""
        N.check(N.lib().b200_dist_cg_start(self._h, C.c_void_p(stream)))

    def step(self, stream: int = 0):
        N.check(N.lib().b200_dist_cg_step(self._h, C.c_void_p(stream)))

    def finish(self, stream: int = 0):
        N.check(N.lib().b200_dist_cg_finish(self._h, C.c_void_p(stream)))

    def scalars(self, stream: int = 0):
        rho, rn = C.c_double(), C.c_double()
        N.check(N.lib().b200_dist_cg_scalars(self._h, C.c_void_p(stream), C.byref(rho), C.byref(rn)))
        return rho.value, rn.value

    def bounds(self):
        b = np.zeros(self.world + 1, np.int64)
        N.check(N.lib().b200_dist_cg_bounds(self._h, N.ptr(b)))
        return b

    def npb(self, niter: int, shift: float):
        z, r = C.c_double(), C.c_double()
        N.check(N.lib().b200_dist_npb(self._h, niter, shift, C.byref(z), C.byref(r)))
        return z.value, r.value

    def info(self, shard: int = 0):
        r0, rows, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        tiled = C.c_int32()
        N.check(N.lib().b200_dist_cg_info(self._h, shard, C.byref(r0), C.byref(rows), C.byref(nnz),
                                          C.byref(tiled)))
        return {"row0": r0.value, "rows": rows.value, "nnz": nnz.value, "tiled": bool(tiled.value)}

    def free(self):
        if self._h:
            N.lib().b200_dist_cg_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def shard_footprint(row_ptr, col_ind):
    """[min col, max col + 1) of a row block's nonzeros (0, 0 when empty)."""
    lo, hi = np.zeros(1, np.int64), np.zeros(1, np.int64)
    N.lib().b200_shard_footprint(len(row_ptr) - 1, N.ptr(row_ptr), N.ptr(col_ind), N.ptr(lo), N.ptr(hi))
    return int(lo[0]), int(hi[0])


def send_ranges(bounds, fmin, fmax):
    """The sharded driver's exchange plan: out[s, r] = [lo, hi) of shard s's
    slice (slice-relative) that rank r reads."""
    world = len(bounds) - 1
    out = np.zeros((world, world, 2), np.int64)
    N.lib().b200_dist_send_ranges(world, N.ptr(np.ascontiguousarray(bounds, np.int64)),
                                  N.ptr(np.ascontiguousarray(fmin, np.int64)),
                                  N.ptr(np.ascontiguousarray(fmax, np.int64)), N.ptr(out.reshape(-1)))
    return out
