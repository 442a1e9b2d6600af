"""Synthetic inputs of the BASELINE.json config shapes, host side.

These are bench/test inputs, not part of the harness path: the matrices a
LiLAC-rewritten program would hand to the entry points. NPB's makea is native
(`device.gen_npb`, C++, bit-identical to the oracle restatement); the 27-point
stencil at full size is generated in HBM (`device.Matrix.stencil27`) and here
only by row range, for CPU checks and baselines.
"""
from __future__ import annotations

import numpy as np

PARBOIL_SEED = 20240817


def gen_parboil(seed: int = PARBOIL_SEED, n: int = 146_000, nnz_target: int = 1_500_000):
    """Parboil SpMV shape (SURVEY §8(d) input 3): row lengths from a clipped
    lognormal (sigma 0.6, 1..64, mean ~ nnz/n), columns uniform in a +-n/8 band
    around the diagonal, ascending per row, values U(-2,2) without 0."""
    rng = np.random.default_rng(seed)
    mean = nnz_target / n
    lens = np.clip(np.round(rng.lognormal(np.log(mean) - 0.18, 0.6, n)), 1, 64).astype(np.int64)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    band = n // 8
    rows = np.repeat(np.arange(n), lens)
    ci = np.clip(rows + rng.integers(-band, band + 1, rp[-1]), 0, n - 1)
    order = np.lexsort((ci, rows))  # ascending columns per row (duplicates allowed)
    ci = ci[order].astype(np.int64)
    val = rng.uniform(-2, 2, rp[-1])
    val[val == 0] = 1.0
    return rp, ci, val


def csr_to_jds(rp, ci, val):
    """The jds_from_dense contract (reference tests/support/oracles.hpp:109-144)
    applied to CSR with ascending columns: rows stable-sorted by nonzero count
    descending (ties keep the original order), perm[orig] = jagged position,
    diagonal k holds the k-th nonzero of every jagged row longer than k."""
    n = len(rp) - 1
    lens = np.diff(rp)
    order = np.argsort(-lens, kind="stable")
    perm = np.empty(n, np.int64)
    perm[order] = np.arange(n)
    nzcnt = lens[order].astype(np.int64)
    max_nz = int(nzcnt[0]) if n else 0
    counts = np.array([(nzcnt > k).sum() for k in range(max_nz)], np.int64)
    jd_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    jval = np.empty(rp[-1], np.float64)
    jcol = np.empty(rp[-1], np.int64)
    starts = rp[order]
    for k in range(max_nz):
        m = counts[k]
        src = starts[:m] + k
        jval[jd_ptr[k]:jd_ptr[k + 1]] = val[src]
        jcol[jd_ptr[k]:jd_ptr[k + 1]] = ci[src]
    return perm, nzcnt, jd_ptr, jval, jcol


def jds_slice(nzcnt, perm, val, jd_ptr, col_ind, j0, j1):
    """The sub-JDS of jagged rows [j0, j1): its own nzcnt / perm / jd_ptr /
    val / col_ind, plus the original row indices it produces (ascending), so
    out[orig_rows] = spmv_jds(sub). Each sub-row keeps its diagonal order, so a
    sliced evaluation is bit-identical to the whole one."""
    sub_nz = np.ascontiguousarray(nzcnt[j0:j1])
    max_nz = int(sub_nz[0]) if len(sub_nz) else 0
    orig = np.nonzero((perm >= j0) & (perm < j1))[0].astype(np.int64)
    sub_perm = (perm[orig] - j0).astype(np.int64)
    counts = np.array([(sub_nz > k).sum() for k in range(max_nz)], np.int64)
    sub_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    sv = np.empty(int(sub_ptr[-1]), np.float64)
    sc = np.empty(int(sub_ptr[-1]), np.int64)
    for k in range(max_nz):
        m = counts[k]
        src = jd_ptr[k] + j0
        sv[sub_ptr[k]:sub_ptr[k + 1]] = val[src:src + m]
        sc[sub_ptr[k]:sub_ptr[k + 1]] = col_ind[src:src + m]
    return sub_nz, sub_perm, sv, sub_ptr, sc, orig


def gen_kronecker(scale: int, edgefactor: int = 16, seed: int = 1, a=0.57, b=0.19, c=0.19):
    """Graph500 Kronecker graph as the PageRank operator (CSR of the transposed,
    column-stochastic adjacency: row = dst, col = src ascending, val =
    1/outdeg(src)), from the native generator (b200_gen_kronecker: counter-based
    hashed uniforms, host threads; scale 22 in seconds)."""
    from . import _native as N
    n = 1 << scale
    m = edgefactor * n
    rp = np.zeros(n + 1, np.int64)
    ci = np.empty(m, np.int64)
    val = np.empty(m, np.float64)
    N.check(N.lib().b200_gen_kronecker(scale, edgefactor, seed, a, b, c, N.ptr(rp), N.ptr(ci), N.ptr(val)))
    return rp, ci, val


def gen_kronecker_reference(scale: int, edgefactor: int = 16, seed: int = 1, a=0.57, b=0.19, c=0.19):
    """Pure-numpy restatement of b200_gen_kronecker (same hashed uniforms,
    same permutation, same CSR build): the CPU check of the native generator
    at small scales."""
    M = (1 << 64) - 1
    n = 1 << scale
    m = edgefactor * n

    def mix(z):
        z = (z + 0x9e3779b97f4a7c15) & M
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M
        return z ^ (z >> 31)

    def unit(e, k):
        return (mix((mix(seed ^ mix(e)) + k) & M) >> 11) * 2.0 ** -53

    ab = a + b
    c_norm, a_norm = c / (1 - ab), a / ab
    src = np.zeros(m, np.int64)
    dst = np.zeros(m, np.int64)
    for e in range(m):
        s = d = 0
        for ib in range(scale):
            ii = int(unit(e, 2 * ib) > ab)
            jj = int(unit(e, 2 * ib + 1) > (c_norm if ii else a_norm))
            s |= ii << ib
            d |= jj << ib
        src[e], dst[e] = s, d
    perm = np.arange(n, dtype=np.int64)
    for i in range(n - 1, 0, -1):
        j = mix((mix(seed ^ 0x5eed) + i) & M) % (i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    src, dst = perm[src], perm[dst]
    outdeg = np.bincount(src, minlength=n).astype(np.float64)
    order = np.lexsort((src, dst))
    src, dst = src[order], dst[order]
    rp = np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))]).astype(np.int64)
    return rp, src.astype(np.int64), 1.0 / outdeg[src]


def stencil27_nnz(nx: int) -> int:
    a = 3 * nx - 2 if nx >= 2 else nx
    return a * a * a


def stencil27_prefix_nnz(nx: int, r: int) -> int:
    """Nonzeros in rows [0, r) of the stencil (csrc/workloads_dev.cu's
    stencil27_prefix_nnz): per axis a point has 1 + (v > 0) + (v < nx - 1)
    neighbours, so a row's count is the product over its three coordinates."""
    def span(v):
        return 1 + (v > 0) + (v < nx - 1)

    def cum(m):  # sum of span(v) for v < m
        return m + max(m - 1, 0) + min(m, nx - 1)
    S = cum(nx)
    i, rem = divmod(r, nx * nx)
    j, k = divmod(rem, nx)
    total = cum(i) * S * S
    if i < nx:
        total += span(i) * (cum(j) * S + span(j) * cum(k))
    return total


def stencil27_bounds(nx: int, k: int):
    """The sharded driver's row bounds (dist_driver.cpp stencil_bounds): shard
    g starts at the first row whose prefix nonzero count reaches
    ceil(nnz * g / k)."""
    n = nx ** 3
    nnz = stencil27_prefix_nnz(nx, n)
    b = [0] * (k + 1)
    for g in range(1, k):
        target = (nnz * g + k - 1) // k
        lo, hi = b[g - 1], n
        while lo < hi:
            mid = (lo + hi) // 2
            if stencil27_prefix_nnz(nx, mid) < target:
                lo = mid + 1
            else:
                hi = mid
        b[g] = lo
    b[k] = n
    return np.array(b, np.int64)


def gen_stencil27_rows(nx: int, r0: int = 0, r1: int | None = None, diag: float = 26.1, offdiag: float = -1.0):
    """Rows [r0, r1) of the 27-point stencil on an nx^3 grid (lexicographic
    rows, neighbours in increasing column order, `diag` on the diagonal): the
    same arrays the device generator (workloads_dev.cu) writes. row_ptr is
    rebased to 0; columns are global."""
    n = nx ** 3
    r1 = n if r1 is None else r1
    idx = np.arange(r0, r1, dtype=np.int64)
    i, j, k = idx // (nx * nx), (idx // nx) % nx, idx % nx
    offs = [(di, dj, dk) for di in (-1, 0, 1) for dj in (-1, 0, 1) for dk in (-1, 0, 1)]
    V = np.stack([(i + di >= 0) & (i + di < nx) & (j + dj >= 0) & (j + dj < nx) & (k + dk >= 0) & (k + dk < nx)
                  for di, dj, dk in offs], axis=1)
    lens = V.sum(axis=1)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    lin = np.array([di * nx * nx + dj * nx + dk for di, dj, dk in offs], np.int64)
    cols = (idx[:, None] + lin[None, :])[V]
    vals = np.broadcast_to(np.where(lin == 0, diag, offdiag), V.shape)[V]
    return rp, cols.astype(np.int64), np.ascontiguousarray(vals, np.float64)


def gen_stencil27(nx: int, diag: float = 26.1, offdiag: float = -1.0):
    return gen_stencil27_rows(nx, 0, nx ** 3, diag, offdiag)


def stencil27_rowsum(nx: int, r0: int, r1: int, diag: float = 26.1, offdiag: float = -1.0):
    """(A 1)[r0:r1] for the stencil: diag + offdiag * (neighbours - 1)."""
    idx = np.arange(r0, r1, dtype=np.int64)
    i, j, k = idx // (nx * nx), (idx // nx) % nx, idx % nx

    def span(v):
        return (v > 0).astype(np.int64) + 1 + (v < nx - 1).astype(np.int64)
    cnt = span(i) * span(j) * span(k)
    return diag + offdiag * (cnt - 1).astype(np.float64)
