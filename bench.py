#!/usr/bin/env python
"""bench.py — B200 benchmark of the LiLAC harness path (BASELINE.json metric).

Workload (N=1 default): NPB CG class C (configs[1] of BASELINE.json): n=150000,
nonzer=15, shift=110, fp64 CSR, matrix resident in HBM, synthetic input from
NPB's own generator (makea). One *step* = one NPB outer iteration = conj_grad
(25 CG steps: fused SpMV+dot, z/r update+dot, p update) + residual SpMV +
norms/x update = 26 SpMVs, captured as one CUDA graph.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0). `value` = NPB iterations/s over the whole job,
device-resident; `e2e` = the same metric through the C-ABI harness entry points
(b200_spmv_csr / b200_dot / b200_axpy / b200_xpay) from pinned host buffers,
i.e. the LiLAC model where the host program keeps its CG loop; `roofline`
= the SpMV kernel's achieved HBM GB/s vs the measured copy peak; `cpu_baseline`
= the reference's own CPU harness (oracle/_ref, interp.cpp:330-389) on a
bounded sample, timed on this box's host cores.
N>1 (torchrun): the row-sharded driver — each rank owns an nnz-balanced row
block, p is all-gathered over NCCL every CG step (strong scaling: the job
advances one NPB iteration per step; value = iterations / max-over-ranks time).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV GFLOP/s & HBM GB/s (% of roofline); NPB-CG iters/sec at 1/2/4/8 B200"
UNIT = "NPB-CG iters/s"
NPB = {  # na, nonzer, niter, shift, zeta_verify (NPB 3.x)
    "S": (1400, 7, 15, 10.0, 8.5971775078648),
    "A": (14000, 11, 15, 20.0, 17.130235054029),
    "B": (75000, 13, 75, 60.0, 22.712745482631),
    "C": (150000, 15, 75, 110.0, 28.973605592845),
}
CGITMAX = 25
SPMV_PER_STEP = CGITMAX + 1


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--npb-class", default="C", choices=sorted(NPB))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--spmv-reps", type=int, default=200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the NPB zeta gate (profiling runs only)")
    ap.add_argument("--no-e2e", action="store_true", help="skip the C-ABI e2e leg (profiling runs only)")
    return ap.parse_args()


def dist_info():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def cpu_desc():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


def cpu_sockets():
    """Distinct physical packages in /proc/cpuinfo (report sockets)."""
    ids = set()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("physical id"):
                    ids.add(line.split(":", 1)[1].strip())
    except OSError:
        pass
    return len(ids) or None


# ------------------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ------------------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "utilization.gpu"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self

        def pump():
            for line in self.proc.stdout:
                self.rows.append([c.strip() for c in line.split(",")])

        self.thread = threading.Thread(target=pump, daemon=True)
        self.thread.start()
        return self

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=1)
        rows = [r for r in self.rows if len(r) == len(self.FIELDS)]
        sm = []
        reasons = set()
        sm_max = None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        loaded = [r for r in rows if _num(r[7]) and _num(r[7]) > 0] or rows
        for r in loaded:
            if _num(r[0]):
                sm.append(_num(r[0]))
            if _num(r[1]):
                sm_max = _num(r[1])
            for k, nm in enumerate(names):
                if r[3 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": sm_max,
                "reasons": sorted(reasons), "samples": len(loaded)}


def _num(s):
    try:
        return float(s)
    except (TypeError, ValueError):
        return None


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_substr: str):
    """Per-launch DRAM bytes of the SpMV kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        for k, v in d.get("kernels", {}).items():
            if kernel_substr in k:
                return v.get("dram_bytes")
    except (OSError, ValueError):
        pass
    return None


# ------------------------------------------------------------------------------------
# reference CPU harness (oracle/_ref) — the baseline arm
# ------------------------------------------------------------------------------------

def host_threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def reference_sample(rp, ci, val, n, reps=1, row_frac=1, threads=None):
    """Times the reference's own HarnessFns ("lilac.spmv_csr" /
    "lilac.dotproduct", interp.cpp:330-389) on `threads` host threads: the
    rows [0, n/row_frac) are cut into nnz-balanced slices, each slice a separate
    HarnessFn call on its own interpreter Memory, run concurrently (the
    interpreter has no shared mutable state; ctypes releases the GIL); the
    dot products likewise by element slices. Returns (seconds per NPB
    iteration, kind, sample description, seconds per full SpMV, threads)."""
    import threading
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    T = threads or host_threads()
    rows_s = max(1, n // row_frac)
    nnz_s = int(rp[rows_s] - rp[0])
    x = np.ones(n)
    bounds = [0]
    for t in range(1, T):
        bounds.append(max(bounds[-1], int(np.searchsorted(rp[: rows_s + 1], rp[0] + nnz_s * t // T))))
    bounds.append(rows_s)
    ebounds = [n * t // T for t in range(T + 1)]
    if O.ref_available():
        R = O.ref()
        kind = "reference"
        keep = []
        hs, hd = [], []
        for t in range(T):
            r0, r1 = bounds[t], bounds[t + 1]
            a, b = int(rp[r0]), int(rp[r1])
            rpt = np.ascontiguousarray(rp[r0:r1 + 1] - rp[r0])
            cit, vt = np.ascontiguousarray(ci[a:b]), np.ascontiguousarray(val[a:b])
            keep += [rpt, cit, vt]
            hs.append(R.ref_prepare_csr(r1 - r0, O.ptr(rpt), O.ptr(vt), O.ptr(x), O.ptr(cit), b - a, n))
            e0, e1 = ebounds[t], ebounds[t + 1]
            xs = np.ascontiguousarray(x[e0:e1])
            keep.append(xs)
            hd.append(R.ref_prepare_dot(e1 - e0, O.ptr(xs), O.ptr(xs)))

        def run(handles):
            th = [threading.Thread(target=lambda h=h: R.ref_call(h)) for h in handles]
            t0 = time.perf_counter()
            for t_ in th:
                t_.start()
            for t_ in th:
                t_.join()
            return time.perf_counter() - t0
    else:
        kind = "port"
        hs = hd = None

        def run(handles):
            t0 = time.perf_counter()
            O.spmv_csr_mt(rp[: rows_s + 1], ci[:nnz_s], val[:nnz_s], x, T) if handles == "spmv" else O.dot(x, x)
            return time.perf_counter() - t0
    t_spmv, t_dot = [], []
    for _ in range(reps):
        t_spmv.append(run(hs if hs is not None else "spmv"))
        t_dot.append(run(hd if hd is not None else "dot"))
    if hs is not None:
        for h in hs + hd:
            R.ref_free(h)
    ts = min(t_spmv) * (int(rp[n] - rp[0]) / max(nnz_s, 1))
    td = min(t_dot)
    dots_per_iter = 2 * CGITMAX + 3
    t_iter = SPMV_PER_STEP * ts + dots_per_iter * td
    desc = (f"{'lilac.spmv_csr/lilac.dotproduct HarnessFns (oracle/_ref)' if kind == 'reference' else 'oracle port'}"
            f" on {T} host threads (nnz-balanced row slices, one interpreter Memory each), rows [0,{rows_s}) "
            f"({nnz_s} nnz) of nnz={int(rp[n] - rp[0])}; x{SPMV_PER_STEP} SpMV + {dots_per_iter} full-length dots "
            f"per NPB iteration; host CG vector updates not counted")
    return t_iter, kind, desc, ts, T


def run_reference(args):
    rank, world, _ = dist_info()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    na, nonzer, niter, shift, _ = NPB[args.npb_class]
    rp, ci, val = O.npb_makea(na, nonzer, shift)
    steps = []
    for i in range(args.warmup + args.steps):
        t_iter, kind, desc, _, threads = reference_sample(rp, ci, val, na, reps=1)
        if i >= args.warmup:
            steps.append(t_iter)
    ms = statistics.mean(steps) * 1e3
    value = 1e3 / ms
    model, ncpu = cpu_desc()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (NPB makea)",
        "config": {"workload": f"NPB CG class {args.npb_class} (n={na}, nnz={int(rp[-1])}) SpMV harness path",
                   "sample": desc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": desc,
                         "cpu": model, "host_cpus": ncpu, "sockets": cpu_sockets()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------

def e2e_harness_cg(rp, ci, val, n, shift, steps, writeback="eager"):
    """NPB outer iterations through the C-ABI harness entry points on pinned
    host vectors (the LiLAC model: host CG loop, offloaded SpMV/dot/axpy).
    writeback="lazy": outputs stay on the device until the host touches them
    (b200_set_writeback; the host-side loop is unchanged)."""
    import torch
    from paper_2001_07938_b200 import harness as H

    H.set_writeback(writeback)
    keep = []

    def pinned(k):
        t = torch.zeros(k + 512, dtype=torch.float64, pin_memory=True)
        keep.append(t)
        a = t.numpy()
        off = (-a.ctypes.data % 4096) // 8  # page-aligned start (lazy write-back needs it)
        return a[off:off + k]

    x, z, r, p, q, res = (pinned(n) for _ in range(6))
    x[:] = 1.0

    def outer():
        z[:] = 0.0
        q[:] = 0.0
        r[:] = x
        p[:] = r
        rho = H.dotproduct(n, r, r)
        for _ in range(CGITMAX):
            H.spmv_csr(n, q, rp, val, p, ci)
            d = H.dotproduct(n, p, q)
            alpha = rho / d
            rho0 = rho
            H.axpy(n, z, alpha, p)
            H.axpy(n, r, -alpha, q)
            rho = H.dotproduct(n, r, r)
            H.xpay(n, p, rho / rho0, r)
        H.spmv_csr(n, r, rp, val, z, ci)
        np.subtract(x, r, out=res)
        rnorm = float(np.sqrt(H.dotproduct(n, res, res)))
        t1 = H.dotproduct(n, x, z)
        t2 = 1.0 / np.sqrt(H.dotproduct(n, z, z))
        x[:] = t2 * z
        return shift + 1.0 / t1, rnorm

    outer()  # first call: uploads the matrix (marshal construct), untimed
    x[:] = 1.0
    st0 = H.harness_stats()
    lz0 = H.lazy_counters()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        zeta, _ = outer()
    t = time.perf_counter() - t0
    st1 = H.harness_stats()
    lz1 = H.lazy_counters()
    H.host_sync()
    H.host_forget()  # the pinned vectors go back to torch's allocator
    H.set_writeback("eager")
    # lazy bytes materialised on host touches are device->host traffic too
    filled = lz1["bytes_filled"] - lz0["bytes_filled"]
    h2d = sum(v["bytes_h2d"] for v in st1.values()) - sum(v["bytes_h2d"] for v in st0.values())
    d2h = sum(v["bytes_d2h"] for v in st1.values()) - sum(v["bytes_d2h"] for v in st0.values())
    calls = sum(v["calls"] for v in st1.values()) - sum(v["calls"] for v in st0.values())
    return {"value": steps / t, "unit": UNIT, "h2d_bytes_per_step": h2d // steps,
            "d2h_bytes_per_step": (d2h + filled) // steps, "harness_calls_per_step": calls // steps,
            "ms_per_step": 1e3 * t / steps, "writeback": writeback,
            "lazy_fills_per_step": (lz1["fault_fills"] + lz1["explicit_fills"] - lz0["fault_fills"]
                                    - lz0["explicit_fills"]) / steps,
            "zeta": zeta,
            "path": "b200_spmv_csr/b200_dot/b200_axpy/b200_xpay on pinned host arrays"}


def e2e_c_host_cg(rp, ci, val, n, shift, steps, writeback="lazy"):
    """NPB outer iterations of a compiled C host program on the harness ABI
    (paper_2001_07938_b200/examples/npb_host_cg.c — conj_grad with its SpMV,
    dot and axpy loops replaced by harness calls, the LiLAC usage model) on
    pinned, page-aligned host vectors."""
    import ctypes as C
    import torch
    from paper_2001_07938_b200 import build as B
    from paper_2001_07938_b200 import harness as H

    E = C.CDLL(B.EX_LIB)
    fn = E.npb_host_cg_outer
    fn.restype = C.c_double
    fn.argtypes = [C.c_int64] + [C.c_void_p] * 9 + [C.c_double, C.POINTER(C.c_double)]
    H.set_writeback(writeback)
    keep = []

    def pinned(k):
        t = torch.zeros(k + 512, dtype=torch.float64, pin_memory=True)
        keep.append(t)
        a = t.numpy()
        off = (-a.ctypes.data % 4096) // 8
        return a[off:off + k]

    x, z, r, p, q, res = (pinned(n) for _ in range(6))
    rn = C.c_double()
    args = [n, rp.ctypes.data, val.ctypes.data, ci.ctypes.data] + [a.ctypes.data for a in (x, z, r, p, q, res)]
    x[:] = 1.0
    fn(*args, shift, C.byref(rn))  # first call: uploads the matrix (marshal construct), untimed
    x[:] = 1.0
    st0 = H.harness_stats()
    lz0 = H.lazy_counters()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        zeta = fn(*args, shift, C.byref(rn))
    t = time.perf_counter() - t0
    st1 = H.harness_stats()
    lz1 = H.lazy_counters()
    H.host_sync()
    H.host_forget()  # the pinned vectors go back to torch's allocator
    H.set_writeback("eager")
    filled = lz1["bytes_filled"] - lz0["bytes_filled"]
    h2d = sum(v["bytes_h2d"] for v in st1.values()) - sum(v["bytes_h2d"] for v in st0.values())
    d2h = sum(v["bytes_d2h"] for v in st1.values()) - sum(v["bytes_d2h"] for v in st0.values())
    calls = sum(v["calls"] for v in st1.values()) - sum(v["calls"] for v in st0.values())
    return {"value": steps / t, "unit": UNIT, "h2d_bytes_per_step": h2d // steps,
            "d2h_bytes_per_step": (d2h + filled) // steps, "harness_calls_per_step": calls // steps,
            "ms_per_step": 1e3 * t / steps, "writeback": writeback, "zeta": zeta, "rnorm": rn.value,
            "path": "C host program (examples/npb_host_cg.c) calling b200_spmv_csr/b200_dot/b200_axpy/b200_xpay "
                    "on pinned host arrays"}


def e2e_dist(cg, shard_rows, shift, steps, stream, world):
    """N > 1: each rank feeds its x slice from pinned host memory, runs one NPB
    outer iteration through the sharded public API (b200_dist_cg_load_x /
    _outer / _result) and reads zeta and rnorm back; max over ranks."""
    import torch
    import torch.distributed as dist
    rows = shard_rows[1] - shard_rows[0]
    x = torch.ones(max(rows, 1), dtype=torch.float64, pin_memory=True)
    sh = stream.cuda_stream

    def step():
        cg.load_x(x.data_ptr(), sh)
        cg.outer(shift, CGITMAX, sh)
        return cg.result()  # synchronises, copies the scalars back

    for _ in range(3):
        step()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    secs = float(t.item())
    return {"value": steps / secs, "unit": UNIT, "h2d_bytes_per_step": 8 * rows * world,
            "d2h_bytes_per_step": 128 * world, "ms_per_step": 1e3 * secs / steps,
            "path": "b200_dist_cg_load_x/_outer/_result per rank (x slice from pinned host, scalars back)"}


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2001_07938_b200 import _native as N
    from paper_2001_07938_b200 import device as D

    rank, world, local = dist_info()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = N.lib()
    N.check(L.b200_init(local))

    na, nonzer, niter, shift, zeta_ref = NPB[args.npb_class]
    t0 = time.perf_counter()
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    t_gen = time.perf_counter() - t0
    nnz = int(rp[-1])
    if world == 1:
        A = D.Matrix.csr(rp, ci, val)
        cg = D.CG(A)
        shard_rows = (0, na)
    else:
        # one shard per rank: nnz-balanced row ranges, NCCL id shared via torch.distributed
        from paper_2001_07938_b200 import dist as PD
        bounds = D.partition_rows(rp, world)
        nid = PD.broadcast_bytes(D.DistCG.nccl_id() if rank == 0 else None, 128, "cuda")
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        cg = D.DistCG.nccl(rank, world, nid, na, bounds, rp[r0:r1 + 1].copy(), ci, val)
        # this rank's row block as a plain resident matrix, for the kernel roofline line
        A = D.Matrix.csr(np.ascontiguousarray(rp[r0:r1 + 1] - rp[r0]), np.ascontiguousarray(ci[rp[r0]:rp[r1]]),
                         np.ascontiguousarray(val[rp[r0]:rp[r1]]))
        shard_rows = (r0, r1)
    info = A.info()

    transport = "single GPU"
    if world > 1:
        transport = "nccl"
        if os.environ.get("LILAC_B200_DIST_P2P", "1") != "0":
            # peer-memory exchange (p2p.cu): kept only if the sharded NPB run
            # verifies on every rank
            from paper_2001_07938_b200 import dist as PD

            def verify():
                zp, _ = cg.npb(niter, shift)
                return abs(zp - zeta_ref) / zeta_ref <= 1e-10

            if PD.attach_peer_memory(cg, verify, "cuda"):
                transport = "p2p"
            else:
                cg.free()
                nid = PD.broadcast_bytes(D.DistCG.nccl_id() if rank == 0 else None, 128, "cuda")
                cg = D.DistCG.nccl(rank, world, nid, na, bounds, rp[r0:r1 + 1].copy(), ci, val)

    # correctness gate: the full NPB benchmark must verify before we time anything
    if args.no_verify:
        zeta, rnorm, verified = None, None, None
    else:
        zeta, rnorm = cg.npb(niter, shift)
        verified = abs(zeta - zeta_ref) / zeta_ref <= 1e-10

    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    cg.reset(sh)
    for _ in range(args.warmup):
        cg.outer(shift, CGITMAX, sh)
    torch.cuda.synchronize()

    clocks = ClockSampler(local).start()
    time.sleep(0.2)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        cg.outer(shift, CGITMAX, sh)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = ev0.elapsed_time(ev1)

    # dominant kernel alone: the CSR SpMV on the same stream, inputs > L2
    x = torch.rand(na, dtype=torch.float64, device="cuda")
    y = torch.empty(max(info["rows"], 1), dtype=torch.float64, device="cuda")
    with torch.cuda.stream(stream):
        for _ in range(5):
            A.spmv(x.data_ptr(), y.data_ptr(), sh)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.spmv_reps):
            A.spmv(x.data_ptr(), y.data_ptr(), sh)
        e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    spmv_ms = e0.elapsed_time(e1) / args.spmv_reps

    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())

    ms_step = ms_total / args.steps
    # strong scaling: the job advances one NPB iteration per step whatever N is
    value = args.steps / (ms_total / 1e3)
    col_b = info["col_bytes"]
    fused_cg = info["kernel"] == 4 and os.environ.get("LILAC_B200_CG_FUSED", "1") != "0"
    snnz, srows = info["nnz"], info["rows"]
    spmv_bytes = snnz * (8 + col_b) + (srows + 1) * 8 + 8 * srows + 8 * info["cols"]
    spmv_flops = 2 * snnz
    peak, peak_src = measured_peak()
    achieved = spmv_bytes / (spmv_ms * 1e-3) / 1e9
    kname = {1: "k_csr_vector", 2: "k_spmv_merge", 3: "k_csr_exact", 4: "k_spmv_tiled", 5: "k_csr_chunks"}.get(info["kernel"], "k_csr_vector")
    traffic = ncu_traffic(kname)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (NPB makea generator, class %s)" % args.npb_class,
        "config": {"workload": f"NPB CG class {args.npb_class}: n={na}, nnz={nnz}, resident CSR "
                               + ("(tiled layout, 16-bit slab-local column keys)" if info["kernel"] == 4
                                  else f"(int{8 * col_b} col_ind)") + f", {SPMV_PER_STEP} SpMV/step",
                   "parallelism": f"row-sharded x{world} ({transport} exchange of p and the dot partials per CG "
                                  "step, CUDA graph per NPB iteration)" if world > 1
                   else "single GPU, CUDA graph per NPB iteration",
                   "shard_rows_rank0": list(shard_rows),
                   "l2": "inputs larger than L2 (matrix %.2f GB > 126 MB)" % (spmv_bytes / 1e9),
                   "zeta": zeta, "zeta_verified": verified, "rnorm": rnorm},
        "cg_iters_per_s": value * CGITMAX,  # CG iterations/s beside NPB outer iterations/s
        "spmv": {"gflops": spmv_flops / (spmv_ms * 1e-3) / 1e9, "gbs": achieved,
                 "frac_of_measured_copy": achieved / peak, "frac_of_nominal_8TBs": achieved / 8000.0,
                 "ms": spmv_ms, "lanes_per_row": info["lanes"], "bytes_per_call": spmv_bytes},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": kname + " (CSR SpMV)",
                     "peak_source": peak_src,
                     "how": f"algorithmic bytes nnz*(8+{col_b})+8(rows+1)+8rows+8cols per launch / mean of "
                            f"{args.spmv_reps} back-to-back launches timed with CUDA events on the bench stream"},
        # per NPB iteration: init, the CG steps (one persistent cooperative kernel on one GPU with the
        # tiled layout, else 3 per step; sharded: 5 per step), residual SpMV + norm, zeta + x update
        "gpu_launches": args.steps * (((1 + 1 + 2 + 2) if fused_cg else (1 + 3 * CGITMAX + 2 + 2)) if world == 1
                                      else (1 + 5 * CGITMAX + 6 + 2)),
        "cg_steps": "one persistent kernel per NPB iteration (grid barriers)" if fused_cg and world == 1
                    else "3 kernels per CG step (programmatic dependent launch)",
        "clocks": clk,
        "gen_s": t_gen,
    }
    if rank == 0 and world == 1 and not args.no_e2e:
        # headline: the compiled C host loop (the LiLAC model) in the faster of
        # the two public write-back modes; the other mode and the Python host
        # loop are reported beside it
        eager = e2e_c_host_cg(rp, ci, val, na, shift, args.e2e_steps, "eager")
        lazy = e2e_c_host_cg(rp, ci, val, na, shift, args.e2e_steps, "lazy")
        line["e2e"], other = (lazy, eager) if lazy["value"] >= eager["value"] else (eager, lazy)
        line["e2e_" + other["writeback"]] = other
        line["e2e_python"] = e2e_harness_cg(rp, ci, val, na, shift, args.e2e_steps, "lazy")
        if not args.no_cpu_baseline:
            t_iter, kind, desc, ts, threads = reference_sample(rp, ci, val, na, reps=2)
            model, ncpu = cpu_desc()
            line["cpu_baseline"] = {"value": 1.0 / t_iter, "unit": UNIT, "cores": threads, "kind": kind,
                                    "sample": desc, "cpu": model, "host_cpus": ncpu, "sockets": cpu_sockets(),
                                    "spmv_s": ts}
    elif world > 1:
        line["e2e"] = e2e_dist(cg, shard_rows, shift, args.e2e_steps * 10, stream, world)
    if rank == 0:
        print(json.dumps(line), flush=True)
    cg.free()
    A.free()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
