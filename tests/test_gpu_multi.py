"""The harness entry points over several GPUs of one process
(LILAC_B200_NGPUS, csrc/multi_harness.cpp), through the unchanged C ABI.

Each case runs in a subprocess (the variable is read once per process). With
fewer GPUs than shards the shards share devices, so on a one-GPU box this
exercises the sharding itself: nnz-balanced row blocks each with its own
resident copy and derived layout, x to every shard, every shard's slice of y
written back, per-shard dot partials summed in order, element-range axpy.
"""
import json
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(code, ngpus):
    env = dict(os.environ, LILAC_B200_NGPUS=str(ngpus))
    r = subprocess.run([sys.executable, "-c", textwrap.dedent(code)], capture_output=True, text=True, timeout=900,
                       cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


PARITY = """
import json, sys
import numpy as np
sys.path.insert(0, "tests")
import oracle_lib as O
from paper_2001_07938_b200 import harness as H, _native as N, device as D
H.set_errors_return(True)
out = {}
rng = np.random.default_rng(5)
n = 60000
lens = rng.integers(0, 40, n)
lens[7] = 30000  # a long row inside one shard
rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
ci = rng.integers(0, n, int(rp[-1])).astype(np.int64)
val = rng.uniform(-2, 2, int(rp[-1]))
x = rng.uniform(-1, 1, n)
y = np.full(n, np.nan)
H.spmv_csr(n, y, rp, val, x, ci)
ref = O.spmv_csr(rp, ci, val, x)
bound = O.spmv_csr(rp, ci, np.abs(val), np.abs(x))
out["spmv"] = bool(np.all(np.abs(y - ref) <= 1e-12 * bound))
x2 = x * 1.5   # a new x (moves); the matrix stays resident
y2 = np.full(n, np.nan)
H.spmv_csr(n, y2, rp, val, x2, ci)
out["spmv_again"] = bool(np.all(np.abs(y2 - O.spmv_csr(rp, ci, val, x2)) <= 1e-12 * 1.5 * bound))
val[100] += 1.0  # the matrix changed: re-sharded
y3 = np.full(n, np.nan)
H.spmv_csr(n, y3, rp, val, x, ci)
out["spmv_changed"] = bool(np.all(np.abs(y3 - O.spmv_csr(rp, ci, val, x))
                                  <= 1e-12 * O.spmv_csr(rp, ci, np.abs(val), np.abs(x))))
a = rng.uniform(-1, 1, 100003)
b = rng.uniform(-1, 1, 100003)
d = H.dotproduct(len(a), a, b)
out["dot"] = bool(abs(d - O.dot(a, b)) <= 1e-12 * O.dot(np.abs(a), np.abs(b)))
yy = b.copy()
H.axpy(len(a), yy, 0.5, a)
out["axpy"] = bool(O.same_bits(yy, O.axpy(b, 0.5, a)))
stats = H.harness_stats()
out["spmv_calls"] = stats["b200_spmv_csr"]["calls"]
print(json.dumps(out))
"""


@pytest.mark.parametrize("ngpus", [2, 3])
def test_multi_gpu_harness_parity(ngpus):
    out = run(PARITY, ngpus)
    for k in ("spmv", "spmv_again", "spmv_changed", "dot", "axpy"):
        assert out[k] is True, (k, out)
    assert out["spmv_calls"] == 3


NPB = """
import ctypes as C, json, sys
import numpy as np
sys.path.insert(0, "tests")
from paper_2001_07938_b200 import build as B, device as D, harness as H
na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES["A"]
rp, ci, val = D.gen_npb(na, nonzer, shift)
E = C.CDLL(B.EX_LIB)
fn = E.npb_host_cg_outer
fn.restype = C.c_double
fn.argtypes = [C.c_int64] + [C.c_void_p] * 9 + [C.c_double, C.POINTER(C.c_double)]
x, z, r, p, q, res = (np.zeros(na) for _ in range(6))
rn = C.c_double()
args = [na, rp.ctypes.data, val.ctypes.data, ci.ctypes.data] + [a.ctypes.data for a in (x, z, r, p, q, res)]
x[:] = 1.0
fn(*args, shift, C.byref(rn))   # NPB's untimed warm-up iteration
x[:] = 1.0
for _ in range(niter):
    zeta = fn(*args, shift, C.byref(rn))
print(json.dumps({"zeta": zeta, "rnorm": rn.value, "ok": abs(zeta - zeta_ref) / zeta_ref <= 1e-10}))
"""


def test_npb_host_cg_class_a_on_two_gpus():
    """examples/npb_host_cg.c (NPB conj_grad with its loops replaced by
    harness calls) unchanged, LILAC_B200_NGPUS=2: zeta verifies."""
    out = run(NPB, 2)
    assert out["ok"] is True, out


PINNED = """
import json, sys
import numpy as np, torch
sys.path.insert(0, "tests")
import oracle_lib as O
from paper_2001_07938_b200 import harness as H, _native as N
H.set_errors_return(True)
n = 20000
rng = np.random.default_rng(8)
lens = rng.integers(1, 20, n)
rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
ci = rng.integers(0, n, int(rp[-1])).astype(np.int64)
val_t = torch.from_numpy(rng.uniform(-1, 1, int(rp[-1]))).pin_memory()
val = val_t.numpy()                 # a pinned input array
x = rng.uniform(-1, 1, n)
y = np.zeros(n)
H.spmv_csr(n, y, rp, val, x, ci)
before = N.lib().b200_dma_visible_regions()
# another library writes the pinned matrix by DMA: no page fault sees it
src = torch.from_numpy(val * 2.0).cuda()
val_t.copy_(src)
torch.cuda.synchronize()
y2 = np.zeros(n)
H.spmv_csr(n, y2, rp, val, x, ci)
ref2 = O.spmv_csr(rp, ci, val, x)
bound = O.spmv_csr(rp, ci, np.abs(val), np.abs(x))
print(json.dumps({"detected": int(before), "fresh": bool(np.all(np.abs(y2 - ref2) <= 1e-12 * bound))}))
"""


def test_pinned_inputs_detected_and_always_policy():
    """A pinned input written by DMA after it was marshaled: the region is
    counted as DMA-visible, and under LILAC_B200_PINNED=always the next call
    re-marshals it (fresh result)."""
    env_old = os.environ.get("LILAC_B200_PINNED")
    os.environ["LILAC_B200_PINNED"] = "always"
    try:
        out = run(PINNED, 1)
    finally:
        if env_old is None:
            os.environ.pop("LILAC_B200_PINNED", None)
        else:
            os.environ["LILAC_B200_PINNED"] = env_old
    assert out["detected"] >= 1 and out["fresh"] is True, out
