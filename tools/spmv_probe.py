"""Kernel probe: times the resident CSR SpMV on NPB class C and on variants of
the same matrix, to separate HBM streaming cost from x-gather (L2) cost.

    python tools/spmv_probe.py [--reps 100] [--only npb]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402


def time_spmv(A, n, reps):
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        A.spmv(x.data_ptr(), y.data_ptr(), s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        A.spmv(x.data_ptr(), y.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def report(name, A, rp, reps):
    n = len(rp) - 1
    nnz = int(rp[-1])
    info = A.info()
    ms = time_spmv(A, n, reps)
    by = nnz * (8 + info["col_bytes"]) + 8 * (n + 1) + 8 * n + 8 * info["cols"]
    kern = {1: "vector", 3: "exact", 4: "tiled"}.get(info["kernel"], "?")
    print(f"{name:28s} {kern:6s} n={n:9d} nnz={nnz:11d} lanes={info['lanes']:2d} {ms*1e3:9.1f} us "
          f"{by/ms/1e6:8.1f} GB/s {2*nnz/ms/1e6:8.1f} GFLOP/s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    N.check(N.lib().b200_init(0))
    rp, ci, val = D.gen_npb(150000, 15, 110.0)
    n = len(rp) - 1
    for kern in (b"vector", b"tiled"):
        N.lib().b200_set_kernel(kern)
        A = D.Matrix.csr(rp, ci, val)
        report("npb_c/" + kern.decode() + "/pf" + os.environ.get("LILAC_B200_TILED_PF", "d"), A, rp, a.reps)
        report("npb_c/" + kern.decode() + "/again", A, rp, a.reps)
        A.free()
    N.lib().b200_set_kernel(b"auto")
    if a.only == "npb":
        return
    # same row structure, columns made local (x gathers hit L1/L2 lines)
    rows = np.repeat(np.arange(n), np.diff(rp))
    lens = np.diff(rp)
    off = np.arange(len(ci)) - np.repeat(rp[:-1], lens)
    ci_local = ((rows + off) % n).astype(np.int64)
    for i in range(0, n, 1):
        pass
    # keep per-row ascending order: rows near the end wrap; sort those rows
    wrap = np.where(rows + lens[rows] > n)[0]
    if len(wrap):
        for r in np.unique(rows[wrap]):
            ci_local[rp[r]:rp[r + 1]].sort()
    A = D.Matrix.csr(rp, ci_local, val)
    report("npb_c_local_cols", A, rp, a.reps)
    A.free()
    # all gathers to one line
    A = D.Matrix.csr(rp, np.zeros_like(ci), val)
    report("npb_c_col0", A, rp, a.reps)
    A.free()
    # 27-nnz rows, random cols over 2M (stencil-ish row length, random gathers)
    n2 = 2_000_000
    rng = np.random.default_rng(0)
    rp2 = (np.arange(n2 + 1) * 27).astype(np.int64)
    ci2 = np.sort(rng.integers(0, n2, (n2, 27)), axis=1).reshape(-1).astype(np.int64)
    v2 = rng.uniform(-1, 1, n2 * 27)
    for kern in (b"vector", b"tiled"):
        N.lib().b200_set_kernel(kern)
        A = D.Matrix.csr(rp2, ci2, v2)
        report("rows27_random/" + kern.decode(), A, rp2, a.reps)
        A.free()
    N.lib().b200_set_kernel(b"auto")
    # banded 27-nnz rows (stencil-like locality)
    ci3 = (np.clip(np.arange(n2)[:, None] + np.arange(-13, 14)[None, :], 0, n2 - 1)).reshape(-1).astype(np.int64)
    A = D.Matrix.csr(rp2, ci3, v2)
    report("rows27_banded", A, rp2, a.reps)
    A.free()


if __name__ == "__main__":
    main()
