#!/usr/bin/env python
"""bench.py — B200 benchmark of the LiLAC harness path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config npb_c|npb_a|parboil|kron|stencil] [--dry-run]

One JSON line per run (rank 0). The default config is BASELINE.json
configs[1], the one the headline metric is quoted on; the others are
configs[0], [2], [3], [4] at their own shapes:

  npb_c    NPB CG class C (n=150000, fp64 CSR from makea); step = one NPB
           outer iteration (25 CG steps + residual = 26 SpMVs + 53 dots);
           unit NPB-CG iters/s. N>1: row-sharded, p exchanged every CG step.
  npb_a    NPB CG class A (n=14000) — the zeta-verification config; the
           reference arm runs the whole benchmark through the reference CPU
           harness (lilac.spmv_csr / lilac.dotproduct HarnessFns).
  parboil  Parboil-shape JDS (n=146000, nnz~1.5M); step = one b200_spmv_jds
           SpMV (L2 flushed between steps: the matrix is L2-sized); GFLOP/s.
  kron     PageRank on a Graph500 Kronecker scale-22 graph (skewed rows);
           step = one power iteration (SpMV + x = 0.85 Ax + 0.15/n); GFLOP/s.
  stencil  27-point stencil N=420 (n=74,088,000, nnz=1,990,865,512), CG on
           A z = A 1; step = one CG iteration; CG iters/s. N>1: row-sharded
           (p halo exchanged every CG step).

Keys beside the contract's: `roofline` (the dominant kernel's algorithmic
bytes per launch / its CUDA-event time, vs MEASURED_PEAKS.json), `e2e` (the
same metric through the C-ABI harness / public API with host buffers, the
copies inside the timed region), `cpu_baseline` (this box's host cores: the
native restatement of the reference semantics at all cores, with one core
and the reference's own HarnessFns beside it), `verify` (results checked in
the cpu_baseline leg against the oracle, or NPB's official zeta).

--gpus N without torchrun re-launches itself under torch.distributed.run with
N ranks (one GPU each, 127.0.0.1 rendezvous). --dry-run runs the N ranks on
CPU over gloo: the product's row partition, footprints and exchange plan
drive a host CG whose exchange follows the device driver's order.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV GFLOP/s & HBM GB/s (% of roofline); NPB-CG iters/sec at 1/2/4/8 B200"
NPB = {  # na, nonzer, niter, shift, zeta_verify (NPB 3.x)
    "S": (1400, 7, 15, 10.0, 8.5971775078648),
    "A": (14000, 11, 15, 20.0, 17.130235054029),
    "B": (75000, 13, 75, 60.0, 22.712745482631),
    "C": (150000, 15, 75, 110.0, 28.973605592845),
}
CGITMAX = 25
SPMV_PER_STEP = CGITMAX + 1
DOTS_PER_STEP = 2 * CGITMAX + 4  # rho0, 2 per CG step, |x - Az|^2, x.z, z.z
STENCIL_NX = 420
KRON_SCALE = 22
DAMPING = 0.85

# one canonical workload string per config: both arms print it (same_config)
WORKLOADS = {
    "npb_c": ("NPB CG class C: n=150000, nonzer=15, shift=110, fp64 CSR from NPB makea; one step = one NPB outer "
              "iteration (25 CG steps + residual: 26 SpMV, 53 dot, CG vector updates)", "NPB-CG iters/s"),
    "npb_a": ("NPB CG class A: n=14000, nonzer=11, shift=20, fp64 CSR from NPB makea; one step = one NPB outer "
              "iteration (26 SpMV, 53 dot, CG vector updates); zeta verified to 1e-10", "NPB-CG iters/s"),
    "parboil": ("Parboil SpMV JDS shape: n=146000, nnz~1.5M (lognormal row lengths sigma 0.6 in 1..64, +-n/8 band, "
                "seed 20240817), fp64 JDS; one step = one spmv_jds", "GFLOP/s"),
    "kron": ("PageRank on Graph500 Kronecker scale 22 (edgefactor 16, seed 1): transposed column-stochastic CSR, "
             "n=4194304; one step = one power iteration (SpMV + x = 0.85 A x + 0.15/n)", "GFLOP/s"),
    "stencil": (f"27-point stencil N={STENCIL_NX}: n={STENCIL_NX ** 3}, nnz=1990865512, diag 26.1 / off -1, fp64 CSR; "
                "CG on A z = A 1 from z = 0; one step = one CG iteration", "CG iters/s"),
}


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="npb_c")
    ap.add_argument("--spmv-reps", type=int, default=200)
    ap.add_argument("--dry-run", action="store_true", help="N ranks on CPU over gloo (no GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the NPB zeta gate (profiling runs only)")
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e legs (profiling runs only)")
    ap.add_argument("--no-scaling-model", action="store_true",
                    help="skip the per-shard SpMV timings (npb_c, stencil at N=1)")
    a = ap.parse_args(argv)
    if a.warmup < 3 and not a.dry_run and a.impl == "ours":
        ap.error("--warmup must be >= 3")
    return a


def dist_info():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args) -> int:
    """--gpus N outside torchrun: one process per GPU under torch.distributed.run."""
    if not args.dry_run:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} requested but {have} GPU(s) visible",
                              "n_gpus": args.gpus}), flush=True)
            return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


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
    ids = set()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("physical id"):
                    ids.add(line.split(":", 1)[1].strip())
    except OSError:
        pass
    return {"cpu": model, "host_cpus": os.cpu_count(), "sockets": len(ids) or None}


def host_threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


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
        time.sleep(0.2)
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
        sm, reasons, sm_max = [], set(), None
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
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_substr: str, config: str):
    """Per-launch DRAM bytes of a kernel from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        for k, v in d.get("kernels", {}).items():
            if kernel_substr in k and v.get("config", "npb_c") == config:
                return v.get("dram_bytes")
    except (OSError, ValueError):
        pass
    return None


def roofline(bytes_per_launch, ms_per_launch, kernel, how, config):
    peak, src = measured_peak()
    achieved = bytes_per_launch / (ms_per_launch * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": ncu_traffic(kernel, config), "kernel": kernel, "peak_source": src, "how": how,
            "frac_of_nominal_8TBs": achieved / 8000.0}


def csr_bytes(info):
    """nnz*(8+s_i) + (rows+1)*8 + 8 rows (y) + 8 cols (x)."""
    return info["nnz"] * (8 + info["col_bytes"]) + 8 * (info["rows"] + 1) + 8 * info["rows"] + 8 * info["cols"]


KERNEL_NAMES = {1: "k_csr_vector", 2: "k_spmv_merge", 3: "k_csr_exact", 4: "k_spmv_tiled", 5: "k_csr_split",
                6: "k_spmv_lrc"}


def base_line(args, config, world, value, ms_step, extra_cfg=None):
    workload, unit = WORKLOADS[config]
    cfg = {"workload": workload, "name": config}
    if extra_cfg:
        cfg.update(extra_cfg)
    return {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg}


# ------------------------------------------------------------------------------------
# CPU legs (oracle: test infrastructure — timed baseline and checker only)
# ------------------------------------------------------------------------------------

def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    return O


def _timed(fn, reps):
    ts = []
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), out


def cpu_npb(rp, ci, val, shift, iters, threads):
    """Native restatement (oracle/oracle.c, what_interp.cpp:87-108 order) of NPB
    outer iterations from x = 1 on `threads` host threads: seconds of the last
    `timed` iterations and the zeta after each iteration."""
    O = _oracle()
    it = O.NpbOuter(rp, ci, val, shift, nthreads=threads)
    zetas, ts = [], []
    for _ in range(iters):
        t0 = time.perf_counter()
        z, _ = it.step()
        ts.append(time.perf_counter() - t0)
        zetas.append(z)
    return ts, zetas


def interp_rate(rp, ci, val, n, threads):
    """The reference's HarnessFn (lilac.spmv_csr, interp.cpp:330-389) on a row
    sample (~2M nonzeros, all threads): seconds per nonzero."""
    O = _oracle()
    if not O.ref_available():
        return None
    target = min(int(rp[n] - rp[0]), 2_000_000)
    r1 = int(np.searchsorted(rp, rp[0] + target))
    r1 = max(1, min(r1, n))
    sub_rp = np.ascontiguousarray(rp[: r1 + 1] - rp[0])
    nz = int(sub_rp[-1])
    A = O.RefCsr(sub_rp, np.ascontiguousarray(ci[rp[0]:rp[0] + nz]), np.ascontiguousarray(val[rp[0]:rp[0] + nz]),
                 int(ci.max()) + 1 if len(ci) else 1, threads)
    x = np.ones(int(ci.max()) + 1 if len(ci) else 1)
    y = np.zeros(r1)
    t, _ = _timed(lambda: A(x, y), 2)
    A.free()
    return t / max(nz, 1)


# ------------------------------------------------------------------------------------
# the reference arm: the reference's own CPU harness, all host threads
# ------------------------------------------------------------------------------------

def run_reference(args):
    rank, world, _ = dist_info()
    if rank != 0:
        return 0
    O = _oracle()
    T = host_threads()
    kind = "reference" if O.ref_available() else "port"
    cfg = args.config
    extra = {}
    if cfg in ("npb_c", "npb_a"):
        cls = "C" if cfg == "npb_c" else "A"
        na, nonzer, niter, shift, zeta_ref = NPB[cls]
        rp, ci, val = O.npb_makea(na, nonzer, shift)
        if kind == "reference":
            cg = O.RefNpbCG(rp, ci, val, shift, T)
            # the interpreter has nothing to warm: a warm-up step is one SpMV + one dot
            for _ in range(args.warmup):
                cg.spmv(cg.p, cg.q)
                cg.dot(cg.p, cg.q)
            steps = []
            zeta = None
            for _ in range(args.steps):
                t0 = time.perf_counter()
                zeta, rnorm = cg.step()
                steps.append(time.perf_counter() - t0)
            sample = (f"{args.steps} full NPB class {cls} outer iterations from x=1 (26 lilac.spmv_csr + 53 "
                      f"lilac.dotproduct HarnessFn calls each, every call split over {T} threads in nnz-balanced "
                      "slices, one interpreter Memory per slice; CG vector updates in numpy); a warm-up step is "
                      "one SpMV + one dot")
            extra["zeta_after_steps"] = zeta
            if cfg == "npb_a":
                # SURVEY §8(d) input 1: the whole benchmark through the reference harness
                cg.x[:] = 1.0
                cg.step()
                cg.x[:] = 1.0
                for _ in range(niter):
                    zeta, rnorm = cg.step()
                extra["npb_zeta"] = zeta
                extra["npb_zeta_verified"] = abs(zeta - zeta_ref) / zeta_ref <= 1e-10
            cg.free()
        else:
            ts, zetas = cpu_npb(rp, ci, val, shift, args.steps, 0)
            steps = ts
            sample = f"{args.steps} NPB class {cls} outer iterations, oracle port on {T} threads"
        ms = statistics.mean(steps) * 1e3
        value = 1e3 / ms
    elif cfg == "parboil":
        from paper_2001_07938_b200 import workloads as W
        rp, ci, val = W.gen_parboil()
        perm, nzcnt, jd_ptr, jval, jcol = W.csr_to_jds(rp, ci, val)
        n, nnz = len(perm), len(jval)
        x = np.random.default_rng(7).uniform(-1, 1, n)
        y = np.zeros(n)
        calls = []
        if kind == "reference":
            # jagged-row slices (bit-identical to the whole call, workloads.jds_slice)
            T_ = min(T, 64)
            bounds = [n * t // T_ for t in range(T_ + 1)]
            keep = []
            R = O.ref()
            for t in range(T_):
                snz, sperm, sv, sptr, sc, orig = W.jds_slice(nzcnt, perm, jval, jd_ptr, jcol, bounds[t],
                                                             bounds[t + 1])
                keep.append((snz, sperm, sv, sptr, sc, orig))
                h = R.ref_prepare_jds(len(snz), O.ptr(snz), O.ptr(sperm), O.ptr(sv), O.ptr(sptr), O.ptr(x), O.ptr(sc),
                                      len(sv), len(sptr), n)
                calls.append((h, orig, np.zeros(len(snz))))

            def one():
                def job(h, orig, out):
                    def f():
                        R.ref_set_floats(h, 6, O.ptr(x), n)
                        R.ref_call(h)
                        R.ref_output(h, O.ptr(out))
                    return f
                O._run_parallel([job(*c) for c in calls])
                for _, orig, out in calls:
                    y[orig] = out
            sample = f"lilac.spmv_jds HarnessFn over {T_} jagged-row slices on {T} threads, one full SpMV per step"
        else:
            def one():
                y[:] = O.spmv_jds_mt(nzcnt, perm, jval, jd_ptr, x, jcol, 0)
            sample = f"oracle port orc_spmv_jds_mt on {T} threads, one full SpMV per step"
        for _ in range(args.warmup):
            one()
        steps = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            one()
            steps.append(time.perf_counter() - t0)
        for c in calls:
            O.ref().ref_free(c[0])
        ms = statistics.mean(steps) * 1e3
        value = 2 * nnz / (ms * 1e-3) / 1e9
    elif cfg == "kron":
        from paper_2001_07938_b200 import workloads as W
        rp, ci, val = W.gen_kronecker(KRON_SCALE)
        n, nnz = len(rp) - 1, len(val)
        x = np.full(n, 1.0 / n)
        y = np.zeros(n)
        if kind == "reference":
            A = O.RefCsr(rp, ci, val, n, T)
            spmv = lambda: A(x, y)  # noqa: E731
            sample = f"lilac.spmv_csr HarnessFn over {T} nnz-balanced row slices; update x = 0.85 y + 0.15/n in numpy"
        else:
            A = None
            spmv = lambda: y.__setitem__(slice(None), O.spmv_csr_mt(rp, ci, val, x, 0))  # noqa: E731
            sample = f"oracle port orc_spmv_csr_mt on {T} threads; numpy update"

        def one():
            spmv()
            np.multiply(y, DAMPING, out=x)
            np.add(x, (1.0 - DAMPING) / n, out=x)
        one()  # a warm-up step (the interpreter has nothing to warm beyond one call)
        steps = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            one()
            steps.append(time.perf_counter() - t0)
        sample += f"; {args.steps} full power iterations timed, 1 warm-up"
        if A is not None:
            A.free()
        ms = statistics.mean(steps) * 1e3
        value = (2 * nnz + 2 * n) / (ms * 1e-3) / 1e9
    else:  # stencil: bounded row sample of one CG iteration, scaled to the full operator
        from paper_2001_07938_b200 import workloads as W
        nx = STENCIL_NX
        n = nx ** 3
        nnz = W.stencil27_nnz(nx)
        frac = 64
        r1 = n // frac
        rp, ci, val = W.gen_stencil27_rows(nx, 0, r1)
        x = np.ones(n)
        y = np.zeros(r1)
        if kind == "reference":
            A = O.RefCsr(rp, ci, val, int(ci.max()) + 1, T)
            spmv = lambda: A(x[: A.ncols], y)  # noqa: E731
            what = "lilac.spmv_csr HarnessFn"
        else:
            A = None
            spmv = lambda: y.__setitem__(slice(None), O.spmv_csr_mt(rp, ci, val, x, 0))  # noqa: E731
            what = "oracle port orc_spmv_csr_mt"
        vn = n // frac
        a, b, c = np.ones(vn), np.ones(vn), np.ones(vn)

        def vec_ops():  # CG vector work of one iteration on the same row sample: 2 dots + 3 axpy-type updates
            float(a @ b)
            np.add(a, 0.5 * b, out=a)
            np.subtract(b, 0.5 * c, out=b)
            float(b @ b)
            np.multiply(c, 0.5, out=c)
            np.add(c, b, out=c)
        spmv()
        vec_ops()
        steps = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            spmv()
            ts = time.perf_counter() - t0
            t0 = time.perf_counter()
            vec_ops()
            steps.append((ts * nnz / rp[-1]) + (time.perf_counter() - t0) * frac)
        if A is not None:
            A.free()
        sample = (f"{what} on rows [0, n/{frac}) ({int(rp[-1])} of {nnz} nonzeros) over {T} threads + the CG vector "
                  f"updates on n/{frac} elements, both scaled to the full operator (extrapolated: a full-size CPU "
                  "iteration does not fit the run)")
        extra["extrapolated"] = True
        ms = statistics.mean(steps) * 1e3
        value = 1e3 / ms
    desc = cpu_desc()
    line = base_line(args, cfg, args.gpus, value, ms, {"sample": sample, **extra})
    line.update({"impl": "reference", "n_gpus": args.gpus,
                 "cpu_baseline": {"value": value, "unit": line["unit"], "cores": T, "kind": kind, "sample": sample,
                                  **desc},
                 "e2e": {"value": value, "unit": line["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------
# our arm, shared pieces
# ------------------------------------------------------------------------------------

class Ctx:
    def __init__(self, args):
        import torch
        import torch.distributed as dist
        from paper_2001_07938_b200 import _native as N
        self.args = args
        self.rank, self.world, self.local = dist_info()
        torch.cuda.set_device(self.local)
        if self.world > 1:
            if torch.cuda.device_count() < self.world:
                raise SystemExit(f"{self.world} ranks but {torch.cuda.device_count()} GPU(s) visible")
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        self.L = N.lib()
        N.check(self.L.b200_init(self.local))
        self.stream = torch.cuda.Stream()
        self.sh = self.stream.cuda_stream

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        if self.world == 1:
            return v
        import torch
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def all_true(self, ok: bool) -> bool:
        if self.world == 1:
            return bool(ok)
        import torch
        import torch.distributed as dist
        t = torch.tensor([1.0 if ok else 0.0], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item() == 1.0)

    def timed_steps(self, step, warmup, steps):
        """W warm-up steps, then K steps between CUDA events on the bench
        stream, barrier + synchronize on both sides; max over ranks (ms)."""
        import torch
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        clocks = ClockSampler(self.local).start()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        self.barrier()
        torch.cuda.synchronize()
        e0.record(self.stream)
        for _ in range(steps):
            step()
        e1.record(self.stream)
        torch.cuda.synchronize()
        self.barrier()
        clk = clocks.stop()
        return self.max_over_ranks(e0.elapsed_time(e1)), clk

    def kernel_ms(self, launch, reps):
        """Mean CUDA-event time of `reps` back-to-back launches on the bench
        stream. A spin kernel ahead of the first event holds the stream until
        every launch is queued, so the host's per-call cost (ctypes, ~10 us)
        never shows up as GPU idle time between small kernels."""
        import torch
        for _ in range(5):
            launch()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(self.stream):
            torch.cuda._sleep(int(2e6) + reps * 40000)  # ~1 ms + 20 us per launch at 1.9 GHz
        e0.record(self.stream)
        for _ in range(reps):
            launch()
        e1.record(self.stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def kernel_ms_cold(self, launch, reps, flush):
        """Mean CUDA-event time of `reps` launches, each after `flush()` (a
        pass over a buffer larger than L2) and bracketed by its own pair of
        events."""
        import torch
        for _ in range(3):
            launch()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        with torch.cuda.stream(self.stream):
            torch.cuda._sleep(int(2e6) + reps * 200000)
            for e0, e1 in ev:
                flush()
                e0.record(self.stream)
                launch()
                e1.record(self.stream)
        torch.cuda.synchronize()
        return sum(e0.elapsed_time(e1) for e0, e1 in ev) / reps

    def finish(self, line):
        if self.rank == 0:
            print(json.dumps(line), flush=True)
        if self.world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return 0


def shard_scaling(ctx, n, full, make_shard, pick, reps, ks=(2, 4, 8)):
    """Kernel-only SpMV scaling of a row-sharded config, measured on this one
    GPU: each shard's row block built as its own resident matrix (the layout
    the sharded driver builds for it) and timed alone over the full x; the
    parallel SpMV time at k GPUs is the slowest shard's. Cold = L2 flushed
    before every launch (the shard's matrix re-read from HBM); warm =
    back-to-back launches (at large k a shard's matrix fits in the 126 MB L2,
    as it would between the CG steps of a real k-GPU run). The flush reads a
    256 MB buffer (a write would leave dirty lines whose write-back lands in
    the timed launch). The p exchange is
    not in these numbers: every gpurun call gets one GPU."""
    import torch
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(11))
    junk = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB > L2
    sink = torch.empty((), dtype=torch.float32, device="cuda")

    def flush():  # a read, not a write: no dirty lines left to write back during the timed launch
        torch.sum(junk, dim=0, out=sink)

    def times(M, rows):
        y = torch.empty(max(rows, 1), dtype=torch.float64, device="cuda")
        f = lambda: M.spmv(x.data_ptr(), y.data_ptr(), ctx.sh)  # noqa: E731
        return ctx.kernel_ms_cold(f, reps, flush), ctx.kernel_ms(f, reps)
    full_cold, full_warm = times(*full)
    out = {"full_ms_cold": full_cold, "full_ms_warm": full_warm, "exchange": "not included (one GPU per run)"}
    for k in ks:
        cold, warm, timed = [], [], list(pick(k))
        for g in timed:
            M, rows = make_shard(k, g)
            c, w = times(M, rows)
            M.free()
            cold.append(c)
            warm.append(w)
        out[str(k)] = {"shards_timed": timed, "max_shard_ms_cold": max(cold), "max_shard_ms_warm": max(warm),
                       "efficiency_cold": full_cold / (k * max(cold)), "efficiency_warm": full_warm / (k * max(warm))}
    del junk, sink
    return out


def harness_bytes(H, st0, st1):
    h2d = sum(v["bytes_h2d"] for v in st1.values()) - sum(v["bytes_h2d"] for v in st0.values())
    d2h = sum(v["bytes_d2h"] for v in st1.values()) - sum(v["bytes_d2h"] for v in st0.values())
    calls = sum(v["calls"] for v in st1.values()) - sum(v["calls"] for v in st0.values())
    return h2d, d2h, calls


# ------------------------------------------------------------------------------------
# NPB CG (configs[0] and [1])
# ------------------------------------------------------------------------------------

def e2e_npb_c_host(rp, ci, val, n, shift, warmup, steps, writeback, memory):
    """NPB outer iterations of a compiled C host program on the harness ABI
    (examples/npb_host_cg.c: conj_grad with its SpMV, dot and axpy loops
    replaced by harness calls — what a LiLAC-rewritten program executes).
    memory = "pinned" (page-aligned pinned vectors) or "pageable" (plain numpy
    arrays, as malloc'd by an unmodified program). The first call marshals the
    matrix (timed separately); then x = 1, W warm-up and K timed iterations.
    Returns the line and the zeta after W+K iterations from x = 1."""
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

    def vec(k):
        if memory == "pageable":
            a = np.zeros(k)
            keep.append(a)
            return a
        t = torch.zeros(k + 512, dtype=torch.float64, pin_memory=True)
        keep.append(t)
        a = t.numpy()
        off = (-a.ctypes.data % 4096) // 8
        return a[off:off + k]

    x, z, r, p, q, res = (vec(n) for _ in range(6))
    rn = C.c_double()
    args_ = [n, rp.ctypes.data, val.ctypes.data, ci.ctypes.data] + [a.ctypes.data for a in (x, z, r, p, q, res)]
    x[:] = 1.0
    t0 = time.perf_counter()
    fn(*args_, shift, C.byref(rn))  # first call: marshals the matrix (construct)
    first_s = time.perf_counter() - t0
    x[:] = 1.0
    for _ in range(warmup):
        fn(*args_, shift, C.byref(rn))
    st0 = H.harness_stats()
    lz0 = H.lazy_counters()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        zeta = fn(*args_, shift, C.byref(rn))
    t = time.perf_counter() - t0
    st1 = H.harness_stats()
    lz1 = H.lazy_counters()
    H.host_sync()
    H.host_forget()
    H.set_writeback("eager")
    h2d, d2h, calls = harness_bytes(H, st0, st1)
    filled = lz1["bytes_filled"] - lz0["bytes_filled"]
    return {"value": steps / t, "unit": "NPB-CG iters/s", "h2d_bytes_per_step": h2d // steps,
            "d2h_bytes_per_step": (d2h + filled) // steps, "harness_calls_per_step": calls // steps,
            "ms_per_step": 1e3 * t / steps, "writeback": writeback, "memory": memory,
            "first_call_s": first_s, "zeta": zeta, "rnorm": rn.value,
            "path": "C host program (examples/npb_host_cg.c) calling b200_spmv_csr/b200_dot/b200_axpy/b200_xpay on "
                    f"{memory} host arrays"}


def e2e_dist(ctx, cg, shard_rows, shift, warmup, steps):
    """N > 1: each rank feeds its x slice from pinned host memory, runs one NPB
    outer iteration through the sharded public API and reads zeta/rnorm back;
    max over ranks."""
    import torch
    rows = shard_rows[1] - shard_rows[0]
    x = torch.ones(max(rows, 1), dtype=torch.float64, pin_memory=True)

    def step():
        cg.load_x(x.data_ptr(), ctx.sh)
        cg.outer(shift, CGITMAX, ctx.sh)
        return cg.result()

    for _ in range(warmup):
        step()
    ctx.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    secs = ctx.max_over_ranks(time.perf_counter() - t0)
    return {"value": steps / secs, "unit": "NPB-CG iters/s", "h2d_bytes_per_step": 8 * rows * ctx.world,
            "d2h_bytes_per_step": 16 * ctx.world, "ms_per_step": 1e3 * secs / steps,
            "path": "b200_dist_cg_load_x/_outer/_result per rank (x slice from pinned host, zeta/rnorm back)"}


def run_npb(ctx, cls):
    import torch
    from paper_2001_07938_b200 import device as D
    args = ctx.args
    cfg = "npb_c" if cls == "C" else "npb_a"
    na, nonzer, niter, shift, zeta_ref = NPB[cls]
    t0 = time.perf_counter()
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    t_gen = time.perf_counter() - t0
    nnz = int(rp[-1])
    transport = "single GPU"
    t0 = time.perf_counter()
    if ctx.world == 1:
        A = D.Matrix.csr(rp, ci, val)
        t_marshal = time.perf_counter() - t0
        cg = D.CG(A)
        shard_rows = (0, na)
    else:
        from paper_2001_07938_b200 import dist as PD
        bounds = D.partition_rows(rp, ctx.world)
        r0, r1 = int(bounds[ctx.rank]), int(bounds[ctx.rank + 1])
        nid = PD.broadcast_bytes(D.DistCG.nccl_id() if ctx.rank == 0 else None, 128, "cuda")
        cg = D.DistCG.nccl(ctx.rank, ctx.world, nid, na, bounds, rp[r0:r1 + 1].copy(), ci, val)
        t_marshal = time.perf_counter() - t0
        A = D.Matrix.csr(np.ascontiguousarray(rp[r0:r1 + 1] - rp[r0]), np.ascontiguousarray(ci[rp[r0]:rp[r1]]),
                         np.ascontiguousarray(val[rp[r0]:rp[r1]]))
        shard_rows = (r0, r1)
        transport = "nccl"
        if os.environ.get("LILAC_B200_DIST_P2P", "1") != "0":
            def verify():
                zp, _ = cg.npb(niter, shift)
                return abs(zp - zeta_ref) / zeta_ref <= 1e-10
            if PD.attach_peer_memory(cg, verify, "cuda"):
                transport = "p2p"
            else:
                cg.free()
                nid = PD.broadcast_bytes(D.DistCG.nccl_id() if ctx.rank == 0 else None, 128, "cuda")
                cg = D.DistCG.nccl(ctx.rank, ctx.world, nid, na, bounds, rp[r0:r1 + 1].copy(), ci, val)
    info = A.info()

    if args.no_verify:
        zeta = rnorm = verified = None
    else:
        zeta, rnorm = cg.npb(niter, shift)
        verified = ctx.all_true(abs(zeta - zeta_ref) / zeta_ref <= 1e-10)

    cg.reset(ctx.sh)
    ms_total, clk = ctx.timed_steps(lambda: cg.outer(shift, CGITMAX, ctx.sh), args.warmup, args.steps)
    ms_step = ms_total / args.steps
    value = args.steps / (ms_total / 1e3)

    # the dominant kernel alone: this rank's SpMV on the same stream, inputs > L2
    x = torch.rand(na, dtype=torch.float64, device="cuda")
    y = torch.empty(max(info["rows"], 1), dtype=torch.float64, device="cuda")
    spmv_ms = ctx.kernel_ms(lambda: A.spmv(x.data_ptr(), y.data_ptr(), ctx.sh), args.spmv_reps)
    by = csr_bytes(info)
    kname = KERNEL_NAMES.get(info["kernel"], "k_csr_vector")
    fused = info["kernel"] == 4 and os.environ.get("LILAC_B200_CG_FUSED", "1") != "0"
    line = base_line(args, cfg, ctx.world, value, ms_step, {
        "matrix": f"n={na}, nnz={nnz}, resident "
                  + ("tiled layout (16-bit slab-local column keys)" if info["kernel"] == 4
                     else f"CSR (int{8 * info['col_bytes']} col_ind)"),
        "parallelism": (f"row-sharded x{ctx.world} ({transport} exchange of p and the dot partials per CG step, "
                        + ("the CG steps in one persistent kernel per GPU (k_cg_tiled_dist), "
                           if ctx.world > 1 and getattr(cg, "fused", False) else "")
                        + "CUDA graph per NPB iteration)") if ctx.world > 1 else "single GPU, CUDA graph per NPB iteration",
        "shard_rows_rank0": list(shard_rows),
        "l2": "inputs larger than L2 (matrix %.2f GB > 126 MB)" % (by / 1e9) if by > 126e6 else
              "matrix smaller than L2 (%.1f MB)" % (by / 1e6),
    })
    line["data"] = f"synthetic (NPB makea generator, class {cls})"
    line["verify"] = {"zeta": zeta, "zeta_ref": zeta_ref, "verified": verified, "rnorm": rnorm,
                      "what": f"full NPB class {cls} benchmark (warm-up + {niter} iterations) on the device path, "
                              "|zeta - official| / official <= 1e-10"}
    line["cg_iters_per_s"] = value * CGITMAX
    line["spmv"] = {"gflops": 2 * info["nnz"] / (spmv_ms * 1e-3) / 1e9, "gbs": by / (spmv_ms * 1e-3) / 1e9,
                    "ms": spmv_ms, "bytes_per_call": by, "kernel": kname}
    line["roofline"] = roofline(by, spmv_ms, kname, f"algorithmic bytes nnz*(8+{info['col_bytes']})+8(rows+1)+8rows+"
                                f"8cols per launch / mean of {args.spmv_reps} back-to-back launches (CUDA events, "
                                "bench stream)", cfg)
    # the whole timed region against the same peak: an NPB iteration's
    # algorithmic bytes (26 SpMV + 25 CG steps' 96n vector bytes + ~48n for
    # the residual and norms) per measured iteration, over all ranks
    pk, _ = measured_peak()
    it_bytes = 26 * by * ctx.world + (25 * 96 + 48) * na
    line["iteration_roofline"] = {"achieved": it_bytes / (ms_step * 1e-3) / 1e9, "peak": pk, "unit": "GB/s",
                                  "frac": it_bytes / (ms_step * 1e-3) / 1e9 / (pk * ctx.world),
                                  "how": "(26 SpMV bytes + (25*96+48) n) per NPB iteration / ms_per_step, "
                                         "peak x n_gpus"}
    dist_fused = ctx.world > 1 and getattr(cg, "fused", False)
    line["gpu_launches"] = args.steps * (((1 + 1 + 2 + 2) if fused else (1 + 3 * CGITMAX + 2 + 2)) if ctx.world == 1
                                         else (4 + 1 + 5 + 3) if dist_fused else (1 + 6 * CGITMAX + 6 + 2))
    line["cg_steps"] = ("one persistent cooperative kernel per NPB iteration (grid barriers)"
                        if fused and ctx.world == 1 else
                        "one persistent kernel per NPB iteration per GPU (shard barriers, peer flags)" if dist_fused
                        else "3 kernels per CG step (programmatic dependent launch)")
    line["clocks"] = clk
    line["marshal_first_call"] = {"s": t_marshal, "h2d_bytes": int(nnz * 16 + (na + 1) * 8),
                                  "device_bytes": info["device_bytes"],
                                  "what": "matrix H2D + validation + int32 narrowing + derived layout build "
                                          "(b200_matrix_create_csr / the sharded driver's shard upload)"}
    line["gen_s"] = t_gen

    if ctx.world == 1 and cls == "C" and not args.no_scaling_model:
        def npb_shard(k, g):
            b = D.partition_rows(rp, k)
            r0, r1 = int(b[g]), int(b[g + 1])
            return D.Matrix.csr(np.ascontiguousarray(rp[r0:r1 + 1] - rp[r0]), np.ascontiguousarray(ci[rp[r0]:rp[r1]]),
                                np.ascontiguousarray(val[rp[r0]:rp[r1]])), r1 - r0
        line["spmv_shard_scaling"] = shard_scaling(ctx, na, (A, na), npb_shard, lambda k: range(k), 20)
    if ctx.world == 1 and not args.no_e2e:
        lazy = e2e_npb_c_host(rp, ci, val, na, shift, args.warmup, args.steps, "lazy", "pinned")
        lazy_pageable = e2e_npb_c_host(rp, ci, val, na, shift, args.warmup, args.steps, "lazy", "pageable")
        eager = e2e_npb_c_host(rp, ci, val, na, shift, args.warmup, args.steps, "eager", "pinned")
        default = e2e_npb_c_host(rp, ci, val, na, shift, args.warmup, args.steps, "eager", "pageable")
        line["e2e"] = lazy
        line["e2e_lazy_pageable"] = lazy_pageable
        line["e2e_eager"] = eager
        line["e2e_default"] = default
        line["e2e"]["note"] = ("headline: pinned page-aligned host vectors with the opt-in lazy write-back "
                               "(b200_set_writeback); e2e_lazy_pageable: plain numpy (malloc'd, adjacent) vectors, "
                               "lazy (an edge page shared with another vector in use is written at once); "
                               "e2e_eager: pinned, eager; e2e_default = the reference semantics an unmodified "
                               "program gets (plain numpy vectors, eager write-back, default strategy)")
    elif ctx.world > 1 and not args.no_e2e:
        line["e2e"] = e2e_dist(ctx, cg, shard_rows, shift, args.warmup, args.steps)

    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        T = host_threads()
        iters = args.warmup + args.steps + (0 if args.no_e2e else 0)
        ts, zetas = cpu_npb(rp, ci, val, shift, args.warmup + args.steps, T)
        t_all = statistics.mean(ts[args.warmup:]) if args.steps else ts[-1]
        ts1, _ = cpu_npb(rp, ci, val, shift, 1, 1)
        rate = interp_rate(rp, ci, val, na, T)
        cb = {"value": 1.0 / t_all, "unit": "NPB-CG iters/s", "cores": T, "kind": "port",
              "sample": (f"native restatement of the reference semantics (oracle/oracle.c orc_npb_outer: "
                         f"what_interp.cpp:87-108 order, -O2 -ffp-contract=off) on {T} threads: {iters} full NPB "
                         f"outer iterations from x=1, the last {args.steps} timed"),
              "one_core": {"value": 1.0 / ts1[0], "sample": "1 thread, 1 full NPB outer iteration"},
              **cpu_desc()}
        if rate is not None:
            spmv_s = rate * nnz
            cb["reference_harness"] = {
                "value": 1.0 / (SPMV_PER_STEP * spmv_s), "ns_per_nnz_all_threads": rate * 1e9,
                "sample": f"lilac.spmv_csr HarnessFn (oracle/_ref) on a ~2M-nonzero row sample over {T} threads; "
                          "value = 1 / (26 SpMV at that rate), dots and vector work not counted"}
        line["cpu_baseline"] = cb
        # the e2e legs' zeta after W+K iterations from x=1, checked against the oracle's
        if "e2e" in line and zetas:
            zref = zetas[-1]
            for k in ("e2e", "e2e_lazy_pageable", "e2e_eager", "e2e_default"):
                z = line[k]["zeta"]
                line[k]["zeta_ref_oracle"] = zref
                line[k]["zeta_verified"] = abs(z - zref) / abs(zref) <= 1e-10
    cg.free()
    A.free()
    return ctx.finish(line)


# ------------------------------------------------------------------------------------
# Parboil-shape JDS (configs[2])
# ------------------------------------------------------------------------------------

def run_parboil(ctx):
    import torch
    from paper_2001_07938_b200 import device as D
    from paper_2001_07938_b200 import harness as H
    from paper_2001_07938_b200 import workloads as W
    args = ctx.args
    t0 = time.perf_counter()
    rp, ci, val = W.gen_parboil()
    perm, nzcnt, jd_ptr, jval, jcol = W.csr_to_jds(rp, ci, val)
    t_gen = time.perf_counter() - t0
    n, nnz, max_nz = len(perm), len(jval), int(nzcnt[0])
    t0 = time.perf_counter()
    A = D.Matrix.jds(nzcnt, perm, jval, jd_ptr, jcol)
    t_marshal = time.perf_counter() - t0
    info = A.info()
    by = (nnz * (8 + info["col_bytes"]) + 16 * n + 8 * (max_nz + 1) + 8 * n + 8 * n)
    xh = np.random.default_rng(7).uniform(-1, 1, n)
    x = torch.from_numpy(xh).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > L2 (126 MB)

    # per step: flush L2 outside the events, time the SpMV alone
    import torch.cuda as tc
    for _ in range(args.warmup):
        A.spmv(x.data_ptr(), y.data_ptr(), ctx.sh)
    torch.cuda.synchronize()
    ev = [(tc.Event(enable_timing=True), tc.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(ctx.local).start()
    ctx.barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(ctx.stream):
        for e0, e1 in ev:
            flush.zero_()
            torch.cuda._sleep(200000)  # holds the stream while the launch is queued (no host gap inside e0..e1)
            e0.record(ctx.stream)
            A.spmv(x.data_ptr(), y.data_ptr(), ctx.sh)
            e1.record(ctx.stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms_total = sum(e0.elapsed_time(e1) for e0, e1 in ev)
    ms_step = ms_total / args.steps
    value = 2 * nnz / (ms_step * 1e-3) / 1e9
    warm_ms = ctx.kernel_ms(lambda: A.spmv(x.data_ptr(), y.data_ptr(), ctx.sh), args.spmv_reps)
    y_dev = y.cpu().numpy()
    line = base_line(args, "parboil", ctx.world, value, ms_step, {
        "l2": "L2 flushed (256 MB write) before every timed step, outside the events; the matrix (%.1f MB) is "
              "otherwise L2-resident" % (by / 1e6),
        "parallelism": "single GPU" if ctx.world == 1 else f"{ctx.world} independent replicas"})
    line["data"] = "synthetic (Parboil-shape generator, seed 20240817)"
    line["spmv"] = {"gflops_cold": value, "gbs_cold": by / (ms_step * 1e-3) / 1e9, "ms_cold": ms_step,
                    "ms_l2_warm": warm_ms, "gflops_l2_warm": 2 * nnz / (warm_ms * 1e-3) / 1e9,
                    "bytes_per_call": by}
    jk = "k_jds_seg" if A.info()["kernel"] == 1 else "k_jds"
    line["spmv"]["kernel"] = jk
    line["roofline"] = roofline(by, ms_step, jk, "JDS algorithmic bytes nnz*(8+s_i)+16 rows+8(max_nz+1)+8 rows+"
                                "8 cols per launch / mean cold-L2 launch time (CUDA events per step)", "parboil")
    line["gpu_launches"] = args.steps
    line["clocks"] = clk
    line["marshal_first_call"] = {"s": t_marshal, "h2d_bytes": int(nnz * 16 + 8 * (2 * n + max_nz + 1)),
                                  "device_bytes": info["device_bytes"]}
    line["gen_s"] = t_gen

    if not args.no_e2e:
        # through the harness entry point: plain numpy arrays, default semantics;
        # x rewritten by the host every step (so it moves), y written back
        H.set_writeback("eager")
        xs = xh.copy()
        ys = np.zeros(n)
        t0 = time.perf_counter()
        H.spmv_jds(n, ys, nzcnt, perm, jval, jd_ptr, xs, jcol)  # first call: marshals the matrix
        first_s = time.perf_counter() - t0
        for i in range(args.warmup):
            np.multiply(xh, 1.0 + 1e-3 * i, out=xs)
            H.spmv_jds(n, ys, nzcnt, perm, jval, jd_ptr, xs, jcol)
        st0 = H.harness_stats()
        t0 = time.perf_counter()
        for i in range(args.steps):
            np.multiply(xh, 1.0 + 1e-3 * i, out=xs)
            H.spmv_jds(n, ys, nzcnt, perm, jval, jd_ptr, xs, jcol)
        t = time.perf_counter() - t0
        st1 = H.harness_stats()
        h2d, d2h, calls = harness_bytes(H, st0, st1)
        line["e2e"] = {"value": 2 * nnz * args.steps / t / 1e9, "unit": "GFLOP/s",
                       "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                       "ms_per_step": 1e3 * t / args.steps, "first_call_s": first_s,
                       "path": "b200_spmv_jds on plain numpy host arrays (eager write-back, default strategy); the "
                               "host rewrites x before every call (x*(1+1e-3 i)), so x moves H2D and y D2H"}
        e2e_x = xs.copy()
        e2e_y = ys.copy()
    if ctx.rank == 0 and not args.no_cpu_baseline:
        O = _oracle()
        T = host_threads()
        t_all, y_ref = _timed(lambda: O.spmv_jds_mt(nzcnt, perm, jval, jd_ptr, xh, jcol, 0), max(3, args.steps))
        t_one, _ = _timed(lambda: O.spmv_jds_mt(nzcnt, perm, jval, jd_ptr, xh, jcol, 1), 2)
        ok = O.same_bits(y_dev, y_ref)
        if not args.no_e2e:
            ok = ok and O.same_bits(e2e_y, O.spmv_jds(nzcnt, perm, jval, jd_ptr, e2e_x, jcol))
        line["verify"] = {"verified": bool(ok), "what": "device and e2e outputs bit-identical to the oracle's "
                                                         "spmv_jds (reference k order)"}
        cb = {"value": 2 * nnz / t_all / 1e9, "unit": "GFLOP/s", "cores": T, "kind": "port",
              "sample": f"native restatement orc_spmv_jds_mt (reference k order) on {T} threads, whole matrix, best of "
                        f"{max(3, args.steps)}",
              "one_core": {"value": 2 * nnz / t_one / 1e9}, **cpu_desc()}
        if O.ref_available():
            R = O.ref()
            h = R.ref_prepare_jds(n, O.ptr(nzcnt), O.ptr(perm), O.ptr(jval), O.ptr(jd_ptr), O.ptr(xh), O.ptr(jcol),
                                  nnz, len(jd_ptr), n)
            t_ref, _ = _timed(lambda: R.ref_call(h), 1)
            yr = np.zeros(n)
            R.ref_output(h, O.ptr(yr))
            R.ref_free(h)
            line["verify"]["reference_harness_bit_identical"] = O.same_bits(y_dev, yr)
            cb["reference_harness"] = {"value": 2 * nnz / t_ref / 1e9,
                                       "sample": "lilac.spmv_jds HarnessFn (oracle/_ref), whole matrix, 1 thread"}
        line["cpu_baseline"] = cb
    A.free()
    return ctx.finish(line)


# ------------------------------------------------------------------------------------
# Kronecker PageRank (configs[3])
# ------------------------------------------------------------------------------------

def run_kron(ctx):
    import torch
    from paper_2001_07938_b200 import device as D
    from paper_2001_07938_b200 import harness as H
    from paper_2001_07938_b200 import workloads as W
    args = ctx.args
    t0 = time.perf_counter()
    rp, ci, val = W.gen_kronecker(KRON_SCALE)
    t_gen = time.perf_counter() - t0
    n, nnz = len(rp) - 1, len(val)
    t0 = time.perf_counter()
    A = D.Matrix.csr(rp, ci, val)
    t_marshal = time.perf_counter() - t0
    info = A.info()
    by = csr_bytes(info)
    x = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    w = torch.empty_like(x)
    nsteps = args.warmup + args.steps
    bufs = [x, w]  # the iterate ping-pongs: step i reads bufs[i % 2] and writes the other

    def pr_step():
        A.pagerank_step(DAMPING, bufs[0].data_ptr(), bufs[1].data_ptr(), ctx.sh)
        bufs.reverse()
    ms_total, clk = ctx.timed_steps(pr_step, args.warmup, args.steps)
    x_dev = bufs[0].cpu().numpy()
    ms_step = ms_total / args.steps
    flops = 2 * nnz + 2 * n
    value = flops / (ms_step * 1e-3) / 1e9
    xr = torch.rand(n, dtype=torch.float64, device="cuda")
    yr = torch.empty_like(xr)
    spmv_ms = ctx.kernel_ms(lambda: A.spmv(xr.data_ptr(), yr.data_ptr(), ctx.sh), max(20, args.spmv_reps // 4))
    kname = KERNEL_NAMES.get(info["kernel"], "k_csr_vector")
    line = base_line(args, "kron", ctx.world, value, ms_step, {
        "l2": "inputs larger than L2 (matrix %.2f GB)" % (by / 1e9),
        "parallelism": "single GPU" if ctx.world == 1 else f"{ctx.world} independent replicas"})
    line["data"] = "synthetic (Graph500 Kronecker generator, scale 22, seed 1)"
    line["pagerank_iters_per_s"] = 1e3 / ms_step
    line["spmv"] = {"gflops": 2 * nnz / (spmv_ms * 1e-3) / 1e9, "gbs": by / (spmv_ms * 1e-3) / 1e9, "ms": spmv_ms,
                    "bytes_per_call": by, "kernel": kname, "max_row": info["max_row"]}
    line["roofline"] = roofline(by, spmv_ms, kname, "CSR algorithmic bytes per launch / mean of back-to-back launches "
                                "(CUDA events, bench stream)", "kron")
    pr_fused = info["kernel"] == 6 and os.environ.get("LILAC_B200_PAGERANK_FUSED", "1") != "0"
    # lane-range: hot gather, main, fix-up (the update folded into the row stores); else SpMV (+ counter reset) + update
    line["gpu_launches"] = args.steps * (3 if pr_fused else {6: 4, 5: 3}.get(info["kernel"], 2))
    line["pagerank_update"] = "fused into the lane-range row stores" if pr_fused else "separate kernel"
    line["clocks"] = clk
    line["marshal_first_call"] = {"s": t_marshal, "h2d_bytes": int(nnz * 16 + (n + 1) * 8),
                                  "device_bytes": info["device_bytes"]}
    line["gen_s"] = t_gen
    if not args.no_e2e:
        H.set_writeback("eager")
        xh = np.full(n, 1.0 / n)
        yh = np.zeros(n)

        def step():
            H.spmv_csr(n, yh, rp, val, xh, ci)
            np.multiply(yh, DAMPING, out=xh)
            xh.__iadd__((1.0 - DAMPING) / n)
        t0 = time.perf_counter()
        step()  # first call marshals the matrix
        first_s = time.perf_counter() - t0
        for _ in range(args.warmup - 1):
            step()
        st0 = H.harness_stats()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        t = time.perf_counter() - t0
        st1 = H.harness_stats()
        h2d, d2h, calls = harness_bytes(H, st0, st1)
        line["e2e"] = {"value": flops * args.steps / t / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d // args.steps,
                       "d2h_bytes_per_step": d2h // args.steps, "ms_per_step": 1e3 * t / args.steps,
                       "first_call_s": first_s,
                       "path": "host PageRank loop: b200_spmv_csr on plain numpy arrays (eager write-back) + the "
                               "x update on the host"}
        x_e2e = xh.copy()
    if ctx.rank == 0 and not args.no_cpu_baseline:
        O = _oracle()
        T = host_threads()
        xc = np.full(n, 1.0 / n)
        ts = []
        for _ in range(nsteps):
            t0 = time.perf_counter()
            yc = O.spmv_csr_mt(rp, ci, val, xc, 0)
            np.multiply(yc, DAMPING, out=xc)
            xc += (1.0 - DAMPING) / n
            ts.append(time.perf_counter() - t0)
        t1c, _ = _timed(lambda: O.spmv_csr_mt(rp, ci, val, xc, 1), 1)
        # PageRank is a contraction: per-step SpMV error <= 1e-12 sum|a||x| stays
        # bounded; 1e-10 relative per element after W+K steps
        err = np.max(np.abs(x_dev - xc) / np.abs(xc))
        ok = err <= 1e-10
        if not args.no_e2e:
            err_e = np.max(np.abs(x_e2e - xc) / np.abs(xc))
            ok = ok and err_e <= 1e-10
        line["verify"] = {"verified": bool(ok), "max_rel_err": float(err),
                          "what": f"x after {nsteps} power iterations from 1/n vs the oracle restatement "
                                  "(orc_spmv_csr_mt + the same update), per element relative <= 1e-10"}
        cb = {"value": flops / statistics.mean(ts[args.warmup:]) / 1e9, "unit": "GFLOP/s", "cores": T,
              "kind": "port", "sample": f"native restatement (orc_spmv_csr_mt + numpy update) on {T} threads, "
                                        f"{nsteps} full power iterations, the last {args.steps} timed",
              "one_core": {"value": 2 * nnz / t1c / 1e9, "sample": "1 thread, one SpMV"}, **cpu_desc()}
        rate = interp_rate(rp, ci, val, n, T)
        if rate is not None:
            cb["reference_harness"] = {"value": 2 / rate / 1e9, "ns_per_nnz_all_threads": rate * 1e9,
                                       "sample": f"lilac.spmv_csr HarnessFn on a ~2M-nonzero row sample, {T} threads"}
        line["cpu_baseline"] = cb
    A.free()
    return ctx.finish(line)


# ------------------------------------------------------------------------------------
# 27-point stencil CG (configs[4])
# ------------------------------------------------------------------------------------

def run_stencil(ctx):
    import torch
    from paper_2001_07938_b200 import device as D
    from paper_2001_07938_b200 import workloads as W
    args = ctx.args
    nx = STENCIL_NX
    n = nx ** 3
    nnz = W.stencil27_nnz(nx)
    t0 = time.perf_counter()
    transport = "single GPU"
    if ctx.world == 1:
        A = D.Matrix.stencil27(nx)
        cg = D.CG(A)
        r0, r1 = 0, n
    else:
        from paper_2001_07938_b200 import dist as PD
        nid = PD.broadcast_bytes(D.DistCG.nccl_id() if ctx.rank == 0 else None, 128, "cuda")
        cg = D.DistCG.stencil27_nccl(ctx.rank, ctx.world, nid, nx)
        transport = "nccl (footprint-limited send/recv)"
        if os.environ.get("LILAC_B200_DIST_P2P", "1") != "0":
            def verify():
                cg.start_rowsum(ctx.sh)
                cg.step(ctx.sh)
                cg.finish(ctx.sh)
                _, rn = cg.scalars(ctx.sh)
                return bool(np.isfinite(rn))
            if PD.attach_peer_memory(cg, verify, "cuda"):
                transport = "p2p (halo pushes over NVLink peer memory)"
            else:
                cg.free()
                nid = PD.broadcast_bytes(D.DistCG.nccl_id() if ctx.rank == 0 else None, 128, "cuda")
                cg = D.DistCG.stencil27_nccl(ctx.rank, ctx.world, nid, nx)
        inf = cg.info(0)
        r0, r1 = inf["row0"], inf["row0"] + inf["rows"]
        A = None
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    rows = r1 - r0
    # b = A 1 (the rows' sums), then CG from z = 0
    if ctx.world == 1:
        ones = torch.ones(n, dtype=torch.float64, device="cuda")
        b = torch.empty_like(ones)
        A.spmv(ones.data_ptr(), b.data_ptr(), ctx.sh)
        torch.cuda.synchronize()
        del ones
        cg.start(b.data_ptr(), ctx.sh)
    else:
        b = None
        cg.start_rowsum(ctx.sh)
    ms_total, clk = ctx.timed_steps(lambda: cg.step(ctx.sh), args.warmup, args.steps)
    ms_step = ms_total / args.steps
    value = 1e3 / ms_step
    cg.finish(ctx.sh)
    rho, rnorm = cg.scalars(ctx.sh)
    bnorm = float(np.sqrt(np.sum(W.stencil27_rowsum(nx, 0, n) ** 2)))
    line = base_line(args, "stencil", ctx.world, value, ms_step, {
        "l2": "inputs larger than L2 (matrix %.1f GB)" % (nnz * 12 / 1e9),
        "parallelism": f"row-sharded x{ctx.world}, {transport}: p halo exchanged every CG step" if ctx.world > 1
                       else "single GPU",
        "rows_rank0": [int(r0), int(r1)]})
    line["data"] = "synthetic (27-point stencil generated in HBM)"
    line["gen_s"] = t_gen
    line["clocks"] = clk
    it_bytes = nnz * 12 + 8 * (n + 1) + 16 * n + 96 * n
    line["cg_iteration"] = {"gbs": it_bytes / (ms_step * 1e-3) / 1e9, "bytes": it_bytes,
                            "frac_of_measured_copy": it_bytes / (ms_step * 1e-3) / 1e9 / measured_peak()[0],
                            "gflops": (2 * nnz + 10 * n) / (ms_step * 1e-3) / 1e9}
    if ctx.world == 1:
        info = A.info()
        by = csr_bytes(info)
        xs = torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
        ys = torch.empty_like(xs)
        spmv_ms = ctx.kernel_ms(lambda: A.spmv(xs.data_ptr(), ys.data_ptr(), ctx.sh), 5)
        kname = KERNEL_NAMES.get(info["kernel"], "k_csr_vector")
        line["spmv"] = {"gflops": 2 * nnz / (spmv_ms * 1e-3) / 1e9, "gbs": by / (spmv_ms * 1e-3) / 1e9,
                        "ms": spmv_ms, "bytes_per_call": by, "kernel": kname}
        line["roofline"] = roofline(by, spmv_ms, kname, "CSR algorithmic bytes (int32 col_ind) per launch / mean of "
                                    "back-to-back launches (CUDA events)", "stencil")
        line["gpu_launches"] = args.steps * 3
        # e2e through the public device API: b from pinned host memory once per
        # timed region, one CG step + its residual scalar read back per step
        if not args.no_e2e:
            bh = torch.from_numpy(W.stencil27_rowsum(nx, 0, n)).pin_memory()
            bd = torch.empty(n, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with torch.cuda.stream(ctx.stream):
                bd.copy_(bh, non_blocking=True)
            cg.start(bd.data_ptr(), ctx.sh)
            for _ in range(args.steps):
                cg.step(ctx.sh)
                cg.scalars(ctx.sh)
            t = time.perf_counter() - t0
            line["e2e"] = {"value": args.steps / t, "unit": "CG iters/s", "h2d_bytes_per_step": 8 * n // args.steps,
                           "d2h_bytes_per_step": 8 * 4, "ms_per_step": 1e3 * t / args.steps,
                           "path": "b200_cg_start (b H2D from pinned host inside the timed region, amortised over "
                                   "the K steps) + per step b200_cg_step and b200_cg_scalars (rho, rnorm to host)"}
            del bd
        ys_h = ys.cpu().numpy()
        xs_h = xs.cpu().numpy()
        if not args.no_scaling_model:
            def st_shard(k, g):
                b = W.stencil27_bounds(nx, k)
                return D.Matrix.stencil27_rows(nx, int(b[g]), int(b[g + 1])), int(b[g + 1] - b[g])
            line["spmv_shard_scaling"] = shard_scaling(ctx, n, (A, n), st_shard, lambda k: (0, k // 2), 3)
    else:
        line["gpu_launches"] = args.steps * (6 + 1)
        if not args.no_e2e:
            # e2e through the sharded public API: each rank's slice of b from
            # pinned host memory (inside the timed region), then per step one
            # CG iteration and the residual scalars back; max over ranks
            bh = torch.from_numpy(W.stencil27_rowsum(nx, r0, r1)).pin_memory()
            ctx.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            cg.load_x(bh.data_ptr(), ctx.sh)
            cg.start(ctx.sh)
            for _ in range(args.steps):
                cg.step(ctx.sh)
                cg.scalars(ctx.sh)
            secs = ctx.max_over_ranks(time.perf_counter() - t0)
            line["e2e"] = {"value": args.steps / secs, "unit": "CG iters/s",
                           "h2d_bytes_per_step": 8 * n // args.steps, "d2h_bytes_per_step": 32 * ctx.world,
                           "ms_per_step": 1e3 * secs / args.steps,
                           "path": "b200_dist_cg_load_x (b slice from pinned host, amortised over the K steps) + "
                                   "b200_dist_cg_start, then per step b200_dist_cg_step + _scalars; max over ranks"}
    line["verify"] = {"rho_recurrence": rho, "rnorm_true": rnorm, "rel_residual": rnorm / bnorm,
                      "what": "true |b - A z| after warm-up + K CG steps beside the recurrence's sqrt(rho)"}
    ok_resid = rnorm / bnorm < 1.0 and abs(rnorm - np.sqrt(max(rho, 0.0))) <= 1e-6 * bnorm
    line["verify"]["verified"] = bool(ctx.all_true(ok_resid))
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        O = _oracle()
        T = host_threads()
        frac = 64
        samples = [(0, n // frac), (n // 2 - n // (2 * frac), n // 2 + n // (2 * frac))]
        ok = True
        t_s, nz_s = 0.0, 0
        for a, e in samples:
            srp, sci, sval = W.gen_stencil27_rows(nx, a, e)
            t, yref = _timed(lambda: O.spmv_csr_mt(srp, sci, sval, xs_h, 0), 2)
            bound = O.spmv_csr_mt(srp, sci, np.abs(sval), np.abs(xs_h), 0)
            ok = ok and bool(np.all(np.abs(ys_h[a:e] - yref) <= 1e-12 * bound))
            t_s += t
            nz_s += int(srp[-1])
        line["verify"]["spmv_rows_checked"] = [list(s) for s in samples]
        line["verify"]["spmv_within_1e-12"] = ok
        line["verify"]["verified"] = bool(line["verify"]["verified"] and ok)
        vn = n // frac
        a_, b_, c_ = np.ones(vn), np.ones(vn), np.ones(vn)

        def vec_ops():
            float(a_ @ b_)
            a_.__iadd__(0.5 * b_)
            b_.__isub__(0.5 * c_)
            float(b_ @ b_)
            c_.__imul__(0.5)
            c_.__iadd__(b_)
        t_v, _ = _timed(vec_ops, 2)
        t_it = t_s * nnz / nz_s + t_v * frac
        cb = {"value": 1.0 / t_it, "unit": "CG iters/s", "cores": T, "kind": "port",
              "sample": f"native restatement orc_spmv_csr_mt on {T} threads over two row samples ({nz_s} of {nnz} "
                        f"nonzeros) + the CG vector updates on n/{frac} elements, scaled to one full CG iteration "
                        "(extrapolated)", **cpu_desc()}
        line["cpu_baseline"] = cb
    cg.free()
    if A is not None:
        A.free()
    return ctx.finish(line)


# ------------------------------------------------------------------------------------
# --dry-run: N CPU ranks over gloo through the product's host-side sharding logic
# ------------------------------------------------------------------------------------

def run_dry(args):
    """The sharded NPB CG on CPU ranks: rows partitioned by the product's
    b200_partition_rows, each rank's footprint by b200_shard_footprint, the p
    exchange following b200_dist_send_ranges (each shard sends each peer only
    the slice range that peer reads), the two dot products gathered and summed
    in rank order — the device driver's sequence (dist_driver.cpp), with host
    arithmetic in place of the kernels."""
    import torch
    import torch.distributed as dist
    from paper_2001_07938_b200 import device as D
    rank, world, _ = dist_info()
    if world > 1:
        dist.init_process_group("gloo")
    stencil = args.config == "stencil"
    cls = "S" if args.config not in ("npb_a",) else "A"
    na, nonzer, niter, shift, zeta_ref = NPB[cls]
    if stencil:  # a 20^3 stencil: banded rows, so the plan is a halo
        from paper_2001_07938_b200 import workloads as W
        nxd = 20
        rp, ci, val = W.gen_stencil27(nxd)
        na = nxd ** 3
    else:
        rp, ci, val = D.gen_npb(na, nonzer, shift)
    bounds = D.partition_rows(rp, world)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    lrp = rp[r0:r1 + 1] - rp[r0]
    lci, lval = ci[rp[r0]:rp[r1]], val[rp[r0]:rp[r1]]
    fmin, fmax = D.shard_footprint(lrp, lci)
    fp = torch.tensor([fmin, fmax], dtype=torch.int64)
    fps = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    if world > 1:
        dist.all_gather(fps, fp)
    else:
        fps = [fp]
    fmins = np.array([int(f[0]) for f in fps])
    fmaxs = np.array([int(f[1]) for f in fps])
    plan = D.send_ranges(bounds, fmins, fmaxs)
    rows_of = np.repeat(np.arange(r1 - r0), np.diff(lrp))

    def spmv(full):
        out = np.zeros(r1 - r0)
        np.add.at(out, rows_of, lval * full[lci])
        return out

    def gather_scalar(v):
        t = torch.tensor([v], dtype=torch.float64)
        if world == 1:
            return v
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, t)
        s = 0.0
        for p_ in parts:  # rank order on every rank
            s += float(p_.item())
        return s

    def exchange(full, mine):
        full[r0:r1] = mine
        if world == 1:
            return
        reqs = []
        for peer in range(world):
            if peer == rank:
                continue
            lo, hi = plan[rank, peer]
            if hi > lo:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(mine[lo:hi])), peer))
        for src in range(world):
            if src == rank:
                continue
            lo, hi = plan[src, rank]
            if hi > lo:
                buf = torch.zeros(int(hi - lo), dtype=torch.float64)
                dist.recv(buf, src)
                full[int(bounds[src]) + lo:int(bounds[src]) + hi] = buf.numpy()
        for r in reqs:
            r.wait()

    x = np.ones(r1 - r0)
    p_full = np.zeros(na)
    z_full = np.zeros(na)

    def outer():
        z = np.zeros(r1 - r0)
        r = x.copy()
        p = r.copy()
        rho = gather_scalar(float(r @ r))
        for _ in range(CGITMAX):
            exchange(p_full, p)
            q = spmv(p_full)
            d = gather_scalar(float(p @ q))
            alpha = rho / d
            rho0 = rho
            z += alpha * p
            r -= alpha * q
            rho = gather_scalar(float(r @ r))
            p = r + (rho / rho0) * p
        exchange(z_full, z)
        res = x - spmv(z_full)
        rn = np.sqrt(gather_scalar(float(res @ res)))
        t1 = gather_scalar(float(x @ z))
        t2 = 1.0 / np.sqrt(gather_scalar(float(z @ z)))
        x[:] = t2 * z
        return shift + 1.0 / t1, rn

    if stencil:
        # plain CG on A z = A 1 from z = 0, 30 iterations; checked against a
        # one-process CG of the same recurrence (whole matrix, numpy)
        ones = np.ones(na)
        x[:] = spmv(ones)  # b = A 1 (own rows)
        iters = 30
        t0 = time.perf_counter()
        z = np.zeros(r1 - r0)
        r = x.copy()
        p = r.copy()
        rho = gather_scalar(float(r @ r))
        for _ in range(iters):
            exchange(p_full, p)
            q = spmv(p_full)
            alpha = rho / gather_scalar(float(p @ q))
            z += alpha * p
            r -= alpha * q
            rho0, rho = rho, gather_scalar(float(r @ r))
            p = r + (rho / rho0) * p
        exchange(z_full, z)
        res = x - spmv(z_full)
        rn = float(np.sqrt(gather_scalar(float(res @ res))))
        secs = time.perf_counter() - t0
        rows_all = np.repeat(np.arange(na), np.diff(rp))

        def spmv_all(v):
            o = np.zeros(na)
            np.add.at(o, rows_all, val * v[ci])
            return o
        b = spmv_all(ones)
        zz, rr = np.zeros(na), b.copy()
        pp = rr.copy()
        rh = float(rr @ rr)
        for _ in range(iters):
            qq = spmv_all(pp)
            al = rh / float(pp @ qq)
            zz += al * pp
            rr -= al * qq
            rh0, rh = rh, float(rr @ rr)
            pp = rr + (rh / rh0) * pp
        rn_ref = float(np.linalg.norm(b - spmv_all(zz)))
        ok = abs(rn - rn_ref) <= 1e-8 * float(np.linalg.norm(b))
        zeta, niter = rn, iters
    else:
        outer()
        x[:] = 1.0
        t0 = time.perf_counter()
        for _ in range(niter):
            zeta, rn = outer()
        secs = time.perf_counter() - t0
        ok = abs(zeta - zeta_ref) / zeta_ref <= 1e-10
    if world > 1:
        t = torch.tensor([1.0 if ok else 0.0])
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ok = bool(t.item() == 1.0)
    if rank == 0:
        print(json.dumps({"dry_run": "gloo", "metric": METRIC, "n_gpus": world, "value": niter / secs,
                          "unit": "NPB-CG iters/s (CPU dry run)", "config": {"workload": "27-point stencil 20^3, 30 CG iterations" if stencil
                                                       else f"NPB CG class {cls}",
                                                                             "bounds": [int(b) for b in bounds]},
                          ("rnorm" if stencil else "zeta"): zeta, "verified": ok,
                          "send_ranges": plan.tolist(), "footprints": [[int(a), int(b)] for a, b in zip(fmins, fmaxs)]}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if ok else 1


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    ctx = Ctx(args)
    if args.config in ("npb_c", "npb_a"):
        return run_npb(ctx, "C" if args.config == "npb_c" else "A")
    if args.config == "parboil":
        return run_parboil(ctx)
    if args.config == "kron":
        return run_kron(ctx)
    return run_stencil(ctx)


if __name__ == "__main__":
    sys.exit(main())
