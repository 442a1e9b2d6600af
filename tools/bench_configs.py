"""Measure every BASELINE.json config shape on one B200 (kernel level).

    python tools/bench_configs.py [--only parboil,kron,stencil,npb] [--stencil-n 256] [--kron-scale 22]

For each config: synthetic input of the named shape, uploaded
once through the resident-device API, then R back-to-back SpMV launches timed
with CUDA events on one stream (inputs larger than L2 except Parboil, which is
L2-resident by construction and reported as such). Prints one JSON line per
config and writes profiles/rNN_configs.md.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402

KERN = {1: "vector", 2: "merge", 3: "exact", 4: "tiled", 5: "split", 0: "jds"}


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def time_spmv(A, n_in, n_out, reps, stream):
    x = torch.rand(n_in, dtype=torch.float64, device="cuda")
    y = torch.empty(max(n_out, 1), dtype=torch.float64, device="cuda")
    for _ in range(5):
        A.spmv(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        A.spmv(x.data_ptr(), y.data_ptr(), stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, x, y


def csr_bytes(info):
    return info["nnz"] * (8 + info["col_bytes"]) + 8 * (info["rows"] + 1) + 8 * info["rows"] + 8 * info["cols"]


def report(name, A, n_in, reps, stream, extra=None, bytes_fn=csr_bytes):
    info = A.info()
    ms, x, y = time_spmv(A, n_in, info["rows"], reps, stream)
    by = bytes_fn(info)
    line = {"config": name, "kernel": KERN.get(info["kernel"], "?") if info["format"] == 0 else "jds",
            "rows": info["rows"], "nnz": info["nnz"], "max_row": info["max_row"], "us": ms * 1e3,
            "gflops": 2 * info["nnz"] / (ms * 1e-3) / 1e9, "gbs": by / (ms * 1e-3) / 1e9,
            "frac_of_measured_copy": by / (ms * 1e-3) / 1e9 / peak(), "bytes_per_call": by}
    if extra:
        line.update(extra)
    print(json.dumps(line), flush=True)
    return line


# ---- generators -------------------------------------------------

def gen_parboil(seed=20240817, n=146_000, nnz_target=1_500_000):
    rng = np.random.default_rng(seed)
    mean = nnz_target / n
    lens = np.clip(np.round(rng.lognormal(np.log(mean) - 0.18, 0.6, n)), 1, 64).astype(np.int64)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    band = n // 8
    rows = np.repeat(np.arange(n), lens)
    ci = np.clip(rows + rng.integers(-band, band + 1, rp[-1]), 0, n - 1)
    # ascending columns per row (duplicates allowed, summed by the math)
    order = np.lexsort((ci, rows))
    ci = ci[order].astype(np.int64)
    val = rng.uniform(-2, 2, rp[-1])
    val[val == 0] = 1.0
    return rp, ci, val


def csr_to_jds(rp, ci, val):
    """jds_from_dense contract (oracles.hpp:109-144) from CSR: stable sort of
    rows by nonzero count descending; perm[orig] = jagged; diagonals."""
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


def gen_kronecker(scale, edgefactor=16, seed=1, a=0.57, b=0.19, c=0.19):
    """Graph500 Kronecker edge list -> CSR of the transposed, column-stochastic
    adjacency (PageRank operator): row = dst, col = src, val = 1/outdeg(src)."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = edgefactor * n
    src = np.zeros(m, np.int64)
    dst = np.zeros(m, np.int64)
    ab = a + b
    c_norm = c / (1 - ab)
    a_norm = a / ab
    for ib in range(scale):
        r1 = rng.random(m)
        r2 = rng.random(m)
        ii = (r1 > ab).astype(np.int64)
        jj = (r2 > (c_norm * ii + a_norm * (1 - ii))).astype(np.int64)
        src += ii << ib
        dst += jj << ib
    # Graph500 permutes vertex labels
    p = rng.permutation(n)
    src, dst = p[src], p[dst]
    outdeg = np.bincount(src, minlength=n).astype(np.float64)
    order = np.lexsort((src, dst))
    src, dst = src[order], dst[order]
    rp = np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))]).astype(np.int64)
    val = 1.0 / outdeg[src]
    return rp, src.astype(np.int64), val


def gen_stencil27(nx):
    """27-point stencil on an nx^3 grid: diag 26.1, off-diag -1 (SPD)."""
    n = nx ** 3
    idx = np.arange(n, dtype=np.int64)
    i, j, k = idx // (nx * nx), (idx // nx) % nx, idx % nx
    offs = [(di, dj, dk) for di in (-1, 0, 1) for dj in (-1, 0, 1) for dk in (-1, 0, 1)]
    valid = []
    for di, dj, dk in offs:
        valid.append((i + di >= 0) & (i + di < nx) & (j + dj >= 0) & (j + dj < nx) & (k + dk >= 0) & (k + dk < nx))
    V = np.stack(valid, axis=1)  # n x 27, offsets in increasing linear order
    lens = V.sum(axis=1)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    lin = np.array([di * nx * nx + dj * nx + dk for di, dj, dk in offs], np.int64)
    cols = (idx[:, None] + lin[None, :])[V]
    vals = np.where(lin[None, :] == 0, 26.1, -1.0) * np.ones((n, 27))
    return rp, cols.astype(np.int64), vals[V]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="parboil,kron,stencil,npb")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--stencil-n", type=int, default=420)
    ap.add_argument("--kron-scale", type=int, default=22)
    ap.add_argument("--round", type=int, default=1)
    a = ap.parse_args()
    N.check(N.lib().b200_init(0))
    stream = torch.cuda.Stream()
    only = a.only.split(",")
    lines = []
    if "npb" in only:
        rp, ci, val = D.gen_npb(150000, 15, 110.0)
        for k in (b"auto", b"vector"):
            N.lib().b200_set_kernel(k)
            A = D.Matrix.csr(rp, ci, val)
            lines.append(report(f"NPB CG class C SpMV ({k.decode()})", A, len(rp) - 1, a.reps, stream))
            A.free()
        N.lib().b200_set_kernel(b"auto")
    if "parboil" in only:
        rp, ci, val = gen_parboil()
        perm, nzcnt, jd_ptr, jval, jcol = csr_to_jds(rp, ci, val)
        A = D.Matrix.jds(nzcnt, perm, jval, jd_ptr, jcol)

        def jds_bytes(info, max_nz=int(nzcnt[0])):
            return (info["nnz"] * (8 + info["col_bytes"]) + 16 * info["rows"] + 8 * (max_nz + 1)
                    + 8 * info["rows"] + 8 * info["cols"])
        lines.append(report("Parboil SpMV JDS shape (n=146k, 1.5M nnz; L2-resident)", A, len(perm), a.reps, stream,
                            bytes_fn=jds_bytes))
        A.free()
        A = D.Matrix.csr(rp, ci, val)
        lines.append(report("Parboil shape as CSR (L2-resident)", A, len(rp) - 1, a.reps, stream))
        A.free()
    if "kron" in only:
        t0 = time.time()
        rp, ci, val = gen_kronecker(a.kron_scale)
        gen_s = time.time() - t0
        A = D.Matrix.csr(rp, ci, val)
        n = len(rp) - 1
        line = report(f"PageRank Kronecker scale {a.kron_scale} (A^T, skewed rows)", A, n, a.reps, stream,
                      extra={"gen_s": gen_s})
        lines.append(line)
        # the workload: 20 PageRank steps (SpMV + x = 0.85 Ax + 0.15/n)
        x = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
        w = torch.empty_like(x)
        A.pagerank(0.85, 2, x.data_ptr(), w.data_ptr(), stream.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()  # the warm-up runs on `stream`; reset x only after it
        x.fill_(1.0 / n)
        torch.cuda.synchronize()
        e0.record(stream)
        A.pagerank(0.85, 20, x.data_ptr(), w.data_ptr(), stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        pr = {"config": f"PageRank Kronecker scale {a.kron_scale}: 20 iterations", "kernel": line["kernel"],
              "rows": n, "nnz": line["nnz"], "max_row": line["max_row"], "us": e0.elapsed_time(e1) * 1e3,
              "gflops": 20 * 2 * line["nnz"] / (e0.elapsed_time(e1) * 1e-3) / 1e9,
              "gbs": 20 * line["bytes_per_call"] / (e0.elapsed_time(e1) * 1e-3) / 1e9,
              "frac_of_measured_copy": 20 * line["bytes_per_call"] / (e0.elapsed_time(e1) * 1e-3) / 1e9 / peak(),
              "bytes_per_call": 20 * line["bytes_per_call"], "sum_x": float(x.sum().item())}
        print(json.dumps(pr), flush=True)
        lines.append(pr)
        A.free()
    if "stencil" in only:
        nx = a.stencil_n
        t0 = time.time()
        A = D.Matrix.stencil27(nx)  # generated in HBM
        torch.cuda.synchronize()
        gen_s = time.time() - t0
        n = nx ** 3
        line = report(f"27-point stencil N={nx} CSR (device-generated)", A, n, max(5, a.reps // 10), stream,
                      extra={"gen_s": gen_s})
        lines.append(line)
        # the workload: 50 CG iterations on A z = A 1 from z = 0
        cg = D.CG(A)
        ones = torch.ones(n, dtype=torch.float64, device="cuda")
        b = torch.empty_like(ones)
        A.spmv(ones.data_ptr(), b.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        cg.solve(b.data_ptr(), 2)
        t0 = time.perf_counter()
        rn = cg.solve(b.data_ptr(), 50)
        dt = time.perf_counter() - t0
        it_bytes = line["bytes_per_call"] + 96 * n
        cgl = {"config": f"27-point stencil N={nx}: CG 50 iterations (b = A*1)", "kernel": line["kernel"],
               "rows": n, "nnz": line["nnz"], "max_row": line["max_row"], "us": dt * 1e6,
               "gflops": 50 * (2 * line["nnz"] + 10 * n) / dt / 1e9, "gbs": 50 * it_bytes / dt / 1e9,
               "frac_of_measured_copy": 50 * it_bytes / dt / 1e9 / peak(), "bytes_per_call": 50 * it_bytes,
               "rnorm_rel": rn / float(torch.linalg.norm(b).item())}
        print(json.dumps(cgl), flush=True)
        lines.append(cgl)
        cg.free()
        A.free()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "configs.jsonl"), "a") as f:
        for ln in lines:
            f.write(json.dumps(ln) + "\n")
    path = os.path.join(ROOT, "gpurun_out", f"r{a.round:02d}_configs.md")
    with open(path, "w") as f:
        f.write(f"# Round {a.round}: SpMV on every BASELINE config shape (1 B200, tools/bench_configs.py)\n\n")
        f.write(f"Peak for the fraction: measured copy {peak():.1f} GB/s (MEASURED_PEAKS.json). Algorithmic bytes "
                "per call per DESIGN.md §5; CUDA events over back-to-back launches on one stream.\n\n")
        f.write("| config | kernel | rows | nnz | max row | us/call | GFLOP/s | GB/s | frac of copy |\n")
        f.write("|---|---|---:|---:|---:|---:|---:|---:|---:|\n")
        for ln in lines:
            f.write(f"| {ln['config']} | {ln['kernel']} | {ln['rows']} | {ln['nnz']} | {ln['max_row']} | "
                    f"{ln['us']:.1f} | {ln['gflops']:.0f} | {ln['gbs']:.0f} | {ln['frac_of_measured_copy']:.3f} |\n")
    print("wrote", path)


if __name__ == "__main__":
    main()
