"""Small cases of every kernel family against the oracle, one process:

    python tools/kernel_smoke.py [csr|tiled|lane|jds|blas|gemm|cg|dist|stencil ...]

(compute-sanitizer is not available on the GPU pool; these small cases with
NaN-filled outputs and oracle comparisons are the substitute.) Families: csr
(vector, split, merge, tiled with 1/2/4 slab parts, lane), jds, blas (dot,
axpy), gemm, cg (fused tiled, per-step), dist (local shards), stencil
(device generator, row block). Exit 1 on a mismatch."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib as O  # noqa: E402
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402
from paper_2001_07938_b200 import harness as H  # noqa: E402
from paper_2001_07938_b200 import workloads as W  # noqa: E402

H.set_errors_return(True)
rng = np.random.default_rng(1)
fails = []


def csr(rows, cols, lens):
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(cols, size=int(k), replace=False)) for k in lens]).astype(np.int64)
    return rp, ci, rng.uniform(-1, 1, int(rp[-1]))


def check(name, ok):
    print(("ok   " if ok else "FAIL ") + name, flush=True)
    if not ok:
        fails.append(name)


def spmv_ok(rp, ci, val, x, y):
    ref = O.spmv_csr(rp, ci, val, x)
    return bool(np.all(np.abs(y - ref) <= 1e-12 * O.spmv_csr(rp, ci, np.abs(val), np.abs(x))))


def fam_csr():
    rows, cols = 6000, 40000
    lens = rng.integers(0, 60, rows)
    lens[5] = 3000
    rp, ci, val = csr(rows, cols, lens)
    x = rng.uniform(-1, 1, cols)
    for k in ("vector", "split", "merge", "lane"):
        N.lib().b200_set_kernel(k.encode())
        y = np.full(rows, np.nan)
        H.spmv_csr(rows, y, rp, val, x, ci)
        check(f"csr {k}", spmv_ok(rp, ci, val, x, y))
    lens = rng.integers(20, 80, rows)
    rp, ci, val = csr(rows, cols, lens)
    for parts in ("1", "2", "4"):
        os.environ["LILAC_B200_TILE_PARTS"] = parts
        N.lib().b200_set_kernel(b"tiled")
        y = np.full(rows, np.nan)
        H.spmv_csr(rows, y, rp, val, x * (1 + int(parts)), ci)
        check(f"csr tiled parts={parts}", spmv_ok(rp, ci, val, x * (1 + int(parts)), y))
    os.environ.pop("LILAC_B200_TILE_PARTS", None)
    N.lib().b200_set_kernel(b"auto")


def fam_jds():
    rp, ci, val = W.gen_parboil(n=3000, nnz_target=30000)
    perm, nzcnt, jd_ptr, jval, jcol = W.csr_to_jds(rp, ci, val)
    x = rng.uniform(-1, 1, 3000)
    y = np.full(3000, np.nan)
    H.spmv_jds(3000, y, nzcnt, perm, jval, jd_ptr, x, jcol)
    check("jds", O.same_bits(y, O.spmv_jds(nzcnt, perm, jval, jd_ptr, x, jcol)))


def fam_blas():
    a, b = rng.uniform(-1, 1, 10001), rng.uniform(-1, 1, 10001)
    d = H.dotproduct(len(a), a, b)
    check("dot", abs(d - O.dot(a, b)) <= 1e-12 * O.dot(np.abs(a), np.abs(b)))
    y = b.copy()
    H.axpy(len(a), y, 0.5, a)
    check("axpy", O.same_bits(y, O.axpy(b, 0.5, a)))


def fam_gemm():
    n, m, p = 70, 45, 33
    a, b = rng.uniform(-1, 1, n * p), rng.uniform(-1, 1, p * m)
    c = np.zeros(n * m)
    H.gemm(n, m, c, p, a, b)
    ref = (a.reshape(n, p) @ b.reshape(p, m)).reshape(-1)
    check("gemm", bool(np.allclose(c, ref, rtol=1e-12, atol=1e-12)))


def fam_cg():
    na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES["S"]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    for k in (b"tiled", b"vector"):
        N.lib().b200_set_kernel(k)
        A = D.Matrix.csr(rp, ci, val)
        cg = D.CG(A)
        zeta, _ = cg.npb(niter, shift)
        check(f"cg {k.decode()}", abs(zeta - zeta_ref) / zeta_ref <= 1e-10)
        cg.free()
        A.free()
    N.lib().b200_set_kernel(b"auto")


def fam_dist():
    na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES["S"]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    d = D.DistCG.local(3, rp, ci, val)
    zeta, _ = d.npb(niter, shift)
    d.free()
    check("dist local x3", abs(zeta - zeta_ref) / zeta_ref <= 1e-10)


def fam_stencil():
    import torch
    nx = 12
    n = nx ** 3
    x = rng.uniform(-1, 1, n)
    xd = torch.from_numpy(x).cuda()
    b = W.stencil27_bounds(nx, 3)
    for pol in (b"auto", b"lane"):
        N.lib().b200_set_kernel(pol)
        M = D.Matrix.stencil27_rows(nx, int(b[1]), int(b[2]))
        y = torch.full((int(b[2] - b[1]),), float("nan"), dtype=torch.float64, device="cuda")
        M.spmv(xd.data_ptr(), y.data_ptr())
        torch.cuda.synchronize()
        M.free()
        srp, sci, sval = W.gen_stencil27_rows(nx, int(b[1]), int(b[2]))
        check(f"stencil rows {pol.decode()}", spmv_ok(srp, sci, sval, x, y.cpu().numpy()))
    N.lib().b200_set_kernel(b"auto")


FAMS = {"csr": fam_csr, "tiled": fam_csr, "lane": fam_stencil, "jds": fam_jds, "blas": fam_blas, "gemm": fam_gemm,
        "cg": fam_cg, "dist": fam_dist, "stencil": fam_stencil}
want = sys.argv[1:] or ["csr", "jds", "blas", "gemm", "cg", "dist", "stencil"]
for f in dict.fromkeys(FAMS[w] for w in want):
    f()
sys.exit(1 if fails else 0)
