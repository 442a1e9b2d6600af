"""Per-harness time breakdown of the C-ABI CG loop (bench e2e leg)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402
from paper_2001_07938_b200 import harness as H  # noqa: E402

N.check(N.lib().b200_init(0))
PROFILE = os.environ.get("DIAG_PROFILE", "1") == "1"
N.lib().b200_set_profiling(1 if PROFILE else 0)
t = time.perf_counter()
for _ in range(100000):
    time.perf_counter_ns()
print("clock read: %.3f us" % ((time.perf_counter() - t) / 100000 * 1e6))
cls = sys.argv[1] if len(sys.argv) > 1 else "C"
mode = sys.argv[2] if len(sys.argv) > 2 else "eager"
na, nonzer, niter, shift, _ = bench.NPB[cls]
rp, ci, val = D.gen_npb(na, nonzer, shift)
N.lib().b200_stats_reset()
import ctypes as C  # noqa: E402
import numpy as np  # noqa: E402


def mc():
    a = np.zeros(4, np.int64)
    N.lib().b200_marshal_counters(N.ptr(a[0:1]), N.ptr(a[1:2]), N.ptr(a[2:3]), N.ptr(a[3:4]))
    return a.copy()


m0 = mc()
t0 = time.perf_counter()
bench.e2e_harness_cg(rp, ci, val, na, shift, int(os.environ.get("DIAG_WARM", "1")), mode)  # warm (matrix upload)
N.lib().b200_stats_reset()
m0 = mc()
r = bench.e2e_harness_cg(rp, ci, val, na, shift, 3, mode)
print("lazy counters", H.lazy_counters())
# Python-side cost of one wrapper call with the C work removed: time the
# argument marshalling (ctypes pointers + error check) alone
x = np.zeros(na)
t = time.perf_counter()
for _ in range(2000):
    N.ptr(x), N.ptr(x), N.ptr(rp), N.ptr(val), N.ptr(ci)
    N.check()
print("ctypes arg marshalling per spmv-shaped call: %.1f us" % ((time.perf_counter() - t) / 2000 * 1e6))
E = H._ext()
bad = np.zeros(na, np.float32)
t = time.perf_counter()
for _ in range(2000):
    try:
        E.axpy(na, bad, 1.0, x)  # rejected at argument checking: binding cost alone
    except TypeError:
        pass
print("binding call + type error per call: %.2f us" % ((time.perf_counter() - t) / 2000 * 1e6))
print("e2e", {k: v for k, v in r.items() if k != "path"})
print("faults, mprotects, hash_bytes, mirror_bytes delta:", (mc() - m0).tolist())
ns = np.zeros(16, np.int64)
cnt = np.zeros(16, np.int64)
k = N.lib().b200_host_profile(N.ptr(ns), N.ptr(cnt), 16)
names = ["mirror_fetch", "mirror_poll", "d2d", "h2d", "d2h+sync", "publish", "publish_guard", "acquire(vec2 in)",
         "launch", "pick(vec2)", "acquire_out(vec2)", "steal", "cudaMalloc"]
for i in range(k):
    print(f"  {names[i]:14s} n={cnt[i]:7d} total={ns[i]/1e6:9.2f} ms mean={ns[i]/max(cnt[i],1)/1e3:8.1f} us")
for name, s in H.harness_stats().items():
    c = max(s["calls"], 1)
    print(f"{name:16s} calls={s['calls']:5d} total/call={1e3*s['t_total_ms']/c:8.1f}us poll={1e3*s['t_poll_ms']/c:8.1f}us "
          f"kernel={1e3*s['t_kernel_ms']/c:8.1f}us wb={1e3*s['t_writeback_ms']/c:8.1f}us "
          f"h2d={s['bytes_h2d']/c/1e6:.2f}MB d2d={s['bytes_d2d']/c/1e6:.2f}MB d2h={s['bytes_d2h']/c/1e6:.2f}MB")
