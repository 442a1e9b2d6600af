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


from paper_2001_07938_b200.workloads import (csr_to_jds, gen_kronecker, gen_parboil,  # noqa: E402,F401
                                              gen_stencil27)


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
