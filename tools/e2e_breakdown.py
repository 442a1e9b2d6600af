"""Per-entry-point host time of the NPB e2e loop (examples/npb_host_cg.c on
the harness ABI): calls, total / poll / kernel / write-back ms per outer
iteration, from b200_harness_stats deltas.

    python tools/e2e_breakdown.py [--cls C] [--writeback lazy|eager] [--memory pinned|pageable] [--steps 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import numpy as np  # noqa: E402

from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402
from paper_2001_07938_b200 import harness as H  # noqa: E402

PHASES = ["mirror_fetch", "mirror_poll", "d2d", "h2d", "d2h+sync", "publish", "publish_guard", "acquire(vec2 in)",
          "launch", "pick(vec2)", "acquire_out(vec2)", "steal", "cudaMalloc"]


def host_profile():
    ns, cnt = np.zeros(16, np.int64), np.zeros(16, np.int64)
    k = N.lib().b200_host_profile(N.ptr(ns), N.ptr(cnt), 16)
    m = np.zeros(4, np.int64)
    N.lib().b200_marshal_counters(N.ptr(m[0:1]), N.ptr(m[1:2]), N.ptr(m[2:3]), N.ptr(m[3:4]))
    return ns[:k].copy(), cnt[:k].copy(), m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cls", default="C")
    ap.add_argument("--writeback", default="lazy")
    ap.add_argument("--memory", default="pinned")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--profile", type=int, default=0, help="1: host phase timers (adds clock reads per call)")
    a = ap.parse_args()
    N.check(N.lib().b200_init(0))
    N.lib().b200_set_profiling(a.profile)
    na, nonzer, niter, shift, _ = D.NPB_CLASSES[a.cls]
    rp, ci, val = D.gen_npb(na, nonzer, shift)
    orig = H.harness_stats
    snaps = []

    profs = []

    def spy():
        s = orig()
        snaps.append(s)
        profs.append(host_profile())
        return s
    H.harness_stats = spy
    line = bench.e2e_npb_c_host(rp, ci, val, na, shift, 3, a.steps, a.writeback, a.memory)
    st0, st1 = snaps[0], snaps[1]
    out = {"ms_per_step": line["ms_per_step"], "value": line["value"]}
    for k in st1:
        d = {f: (st1[k][f] - st0[k][f]) / a.steps for f in ("calls", "t_total_ms", "t_poll_ms", "t_kernel_ms",
                                                            "t_writeback_ms", "bytes_h2d", "bytes_d2h")}
        if d["calls"]:
            out[k] = d
    (ns0, c0, m0), (ns1, c1, m1) = profs[0], profs[1]
    out["host_phases_us_per_step"] = {PHASES[i]: [int(c1[i] - c0[i]) // a.steps, round((ns1[i] - ns0[i]) / 1e3 / a.steps, 1)]
                                      for i in range(len(ns1)) if c1[i] != c0[i]}
    out["faults_mprotects_hashbytes_mirrorbytes_per_step"] = ((m1 - m0) // a.steps).tolist()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
