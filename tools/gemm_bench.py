"""The dense gemm harness kernels on device buffers: the
DMMA kernel (mma.sync m8n8k4 f64) and the exact reference-order kernel,
beside cuBLAS DGEMM (torch.matmul, f64), at square sizes. CUDA events over
back-to-back launches; results checked against cuBLAS (1e-12 relative to
sum |a||b|).

    python tools/gemm_bench.py [--sizes 1024,2048,4096] [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(2e6))
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1024,2048,4096")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--exact-max", type=int, default=2048, help="largest size for the (slow) exact kernel")
    a = ap.parse_args()
    N.check(N.lib().b200_init(0))
    g = torch.Generator("cuda").manual_seed(3)
    for s in (int(v) for v in a.sizes.split(",")):
        A = torch.rand(s, s, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        B = torch.rand(s, s, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        C = torch.empty(s, s, dtype=torch.float64, device="cuda")
        flops = 2.0 * s * s * s
        ref = A @ B
        bound = A.abs() @ B.abs()
        out = {"n": s}
        ms = timed(lambda: D.gemm(s, s, s, A.data_ptr(), B.data_ptr(), C.data_ptr()), a.reps)
        out["dmma_tflops"] = flops / (ms * 1e-3) / 1e12
        out["dmma_ok"] = bool(((C - ref).abs() <= 1e-12 * bound).all())
        ms = timed(lambda: torch.matmul(A, B, out=C), a.reps)
        out["cublas_tflops"] = flops / (ms * 1e-3) / 1e12
        if s <= a.exact_max:
            ms = timed(lambda: D.gemm(s, s, s, A.data_ptr(), B.data_ptr(), C.data_ptr(), exact=True), 2)
            out["exact_tflops"] = flops / (ms * 1e-3) / 1e12
            out["exact_ok"] = bool(((C - ref).abs() <= 1e-12 * bound).all())
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
