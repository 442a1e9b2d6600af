"""Time the CSR kernels on a config matrix (kernel-level, CUDA events, 1 GPU).

    python tools/kernel_sweep.py [--matrix kron|npb_c|parboil_csr|stencil] [--kernels split,lane,...] [--reps 50]

One JSON line per kernel: us per launch, GB/s at the kernel's algorithmic
bytes, fraction of the measured copy peak. LILAC_B200_LRC_HOT caps the
lane-range layout's shared-memory hot set (0 = none)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402
from paper_2001_07938_b200 import workloads as W  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--matrix", default="kron")
    ap.add_argument("--kernels", default="split,lane")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--shard", default="1:0", help="k:g = row block g of the k-way nnz-balanced partition")
    a = ap.parse_args()
    N.check(N.lib().b200_init(0))
    if a.matrix == "kron":
        rp, ci, val = W.gen_kronecker(a.scale)
    elif a.matrix == "npb_c":
        rp, ci, val = D.gen_npb(150000, 15, 110.0)
    elif a.matrix == "parboil_csr":
        rp, ci, val = W.gen_parboil()
    else:
        rp, ci, val = W.gen_stencil27(128)
    cols = int(ci.max()) + 1
    k, g = (int(v) for v in a.shard.split(":"))
    if k > 1:
        b = D.partition_rows(rp, k)
        r0, r1 = int(b[g]), int(b[g + 1])
        rp, ci, val = (np.ascontiguousarray(rp[r0:r1 + 1] - rp[r0]), np.ascontiguousarray(ci[rp[r0]:rp[r1]]),
                       np.ascontiguousarray(val[rp[r0]:rp[r1]]))
    n = len(rp) - 1
    s = torch.cuda.Stream()
    x = torch.rand(cols, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    xh = x.cpu().numpy()
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    ref = O.spmv_csr_mt(rp, ci, val, xh, 0)
    bound = O.spmv_csr_mt(rp, ci, np.abs(val), np.abs(xh), 0)
    for k in a.kernels.split(","):
        N.lib().b200_set_kernel(k.encode())
        A = D.Matrix.csr(rp, ci, val)
        info = A.info()
        for _ in range(3):
            A.spmv(x.data_ptr(), y.data_ptr(), s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            torch.cuda._sleep(int(2e6) + a.reps * 40000)  # queue every launch before the first event
        e0.record(s)
        for _ in range(a.reps):
            A.spmv(x.data_ptr(), y.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        by = info["nnz"] * (8 + info["col_bytes"]) + 8 * (info["rows"] + 1) + 16 * info["rows"]
        ok = bool(np.all(np.abs(y.cpu().numpy() - ref) <= 1e-12 * bound))
        print(json.dumps({"matrix": a.matrix, "shard": a.shard, "requested": k, "kernel": info["kernel"], "us": ms * 1e3,
                          "gbs": by / (ms * 1e-3) / 1e9, "frac": by / (ms * 1e-3) / 1e9 / peak(), "ok": ok,
                          "device_bytes": info["device_bytes"], "hot_env": os.environ.get("LILAC_B200_LRC_HOT")}),
              flush=True)
        A.free()


if __name__ == "__main__":
    main()
