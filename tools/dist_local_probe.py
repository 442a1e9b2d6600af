"""Outer-iteration time of the sharded CG driver with k shards on one GPU
(LocalExchange), e.g. to compare LILAC_B200_DIST_GRAPH=0/1.
    python tools/dist_local_probe.py [k] [class]
DIST_P2P=1: peer-memory exchange; DIST_FUSED=0: its per-step kernels instead of
the persistent sharded CG kernel."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07938_b200 import _native as N  # noqa: E402
from paper_2001_07938_b200 import device as D  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cls = sys.argv[2] if len(sys.argv) > 2 else "C"
na, nonzer, niter, shift, zref = D.NPB_CLASSES[cls]
N.check(N.lib().b200_init(0))
rp, ci, val = D.gen_npb(na, nonzer, shift)
d = D.DistCG.local(k, rp, ci, val)
if os.environ.get("DIST_P2P", "0") == "1":
    d.use_p2p_local()
    d.set_fused(os.environ.get("DIST_FUSED", "1") == "1")
s = torch.cuda.Stream()
d.reset(s.cuda_stream)
for _ in range(3):
    d.outer(shift, 25, s.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record(s)
for _ in range(10):
    d.outer(shift, 25, s.cuda_stream)
e1.record(s)
host = (time.perf_counter() - t0) / 10
torch.cuda.synchronize()
print(f"k={k} class {cls} transport={d.transport} fused={d.fused} graph={os.environ.get('LILAC_B200_DIST_GRAPH', '1')}: "
      f"{e0.elapsed_time(e1) / 10:.3f} ms/outer (host issue {host * 1e3:.3f} ms)")
