"""CPU, world_size 2 (gloo): the row-sharded CG decomposition of the
multi-GPU driver (paper_2001_07938_b200/csrc/dist_driver.cpp), restated with
numpy + the oracle SpMV per shard and torch.distributed for the one exchange
step (all-gather of the p slices, rank-ordered gather of dot partials).

Checks, per rank: the nnz-balanced partition the product computes
(b200_partition_rows) is bit-exact with the oracle's; the sharded NPB CG
verifies zeta and matches the unsharded oracle CG to 1e-12.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def sharded_npb(rank, world, rp, ci, val, bounds, niter, shift):
    n = len(rp) - 1
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    lrp = rp[r0:r1 + 1] - rp[r0]
    lci = ci[rp[r0]:rp[r1]]
    lval = val[rp[r0]:rp[r1]]
    rows = r1 - r0

    def gather_scalars(parts):
        t = torch.tensor(parts, dtype=torch.float64)
        out = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return np.stack([o.numpy() for o in out])  # rank order

    def all_gather_vec(full, own):
        sizes = [int(bounds[g + 1] - bounds[g]) for g in range(world)]
        m = max(sizes)
        t = torch.zeros(m, dtype=torch.float64)
        t[:rows] = torch.from_numpy(own)
        out = [torch.zeros(m, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, t)
        for g in range(world):
            full[bounds[g]:bounds[g + 1]] = out[g].numpy()[:sizes[g]]

    x = np.ones(rows)
    p_full = np.zeros(n)
    z_full = np.zeros(n)
    zeta = rnorm = 0.0
    for it in range(niter + 1):
        z = np.zeros(rows)
        r = x.copy()
        p = r.copy()
        rho = gather_scalars([O.dot(r, r)]).sum(axis=0)[0]
        all_gather_vec(p_full, p)
        for _ in range(25):
            q = O.spmv_csr(lrp, lci, lval, p_full)
            d = gather_scalars([O.dot(p, q)]).sum(axis=0)[0]
            alpha = rho / d
            rho0 = rho
            z = z + alpha * p
            r = r - alpha * q
            rho = gather_scalars([O.dot(r, r)]).sum(axis=0)[0]
            beta = rho / rho0
            p = r + beta * p
            all_gather_vec(p_full, p)
        all_gather_vec(z_full, z)
        rr = O.spmv_csr(lrp, lci, lval, z_full)
        dd = x - rr
        rnorm = np.sqrt(gather_scalars([O.dot(dd, dd)]).sum(axis=0)[0])
        tt = gather_scalars([O.dot(x, z), O.dot(z, z)]).sum(axis=0)
        t2 = 1.0 / np.sqrt(tt[1])
        if it > 0:
            zeta = shift + 1.0 / tt[0]
        x = t2 * z if it > 0 else np.ones(rows)
    return zeta, rnorm


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2001_07938_b200 import device as D
        na, nonzer, niter, shift, zeta_ref = D.NPB_CLASSES["S"]
        rp, ci, val = D.gen_npb(na, nonzer, shift)
        bounds = D.partition_rows(rp, world)
        assert np.array_equal(bounds, O.partition_rows(rp, world))
        zeta, rnorm = sharded_npb(rank, world, rp, ci, val, bounds, niter, shift)
        q.put((rank, zeta, rnorm, bounds.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_cg_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    zetas = {r: z for r, z, _, _ in res}
    # every rank finalised the same scalars in the same order
    assert len(set(zetas.values())) == 1
    zeta = zetas[0]
    assert abs(zeta - 8.5971775078648) / 8.5971775078648 <= 1e-10
    rp, ci, val = O.npb_makea(1400, 7, 10.0)
    z1, _ = O.npb_cg(rp, ci, val, 15, 10.0)
    assert abs(zeta - z1) <= 1e-12 * abs(z1)


# ---- the cross-process handshake of the peer-memory exchange (dist.py) ----------

class _FakeCG:
    """Stands in for DistCG: a rank-specific 208-byte record; remembers what
    p2p_attach received."""

    def __init__(self, rank, fail_attach=False):
        self.record = bytes([rank + 1]) * 200 + rank.to_bytes(8, "little")
        self.got = None
        self.fail_attach = fail_attach

    def p2p_export(self):
        return self.record

    def p2p_attach(self, blob):
        if self.fail_attach:
            raise RuntimeError("no peer access")
        self.got = blob


def _handshake_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2001_07938_b200 import dist as PD
    out = {}
    out["bcast"] = PD.broadcast_bytes(b"nccl-id-" + bytes(120) if rank == 0 else None, 128, "cpu")
    cg = _FakeCG(rank)
    out["kept"] = PD.attach_peer_memory(cg, lambda: True, "cpu")
    out["blob"] = cg.got
    # one rank's verification fails: nobody keeps it
    out["kept_when_one_fails"] = PD.attach_peer_memory(_FakeCG(rank), lambda: rank == 0, "cpu")
    # one rank cannot map its peers: nobody keeps it, no exception escapes
    out["kept_when_attach_fails"] = PD.attach_peer_memory(_FakeCG(rank, fail_attach=rank == 1), lambda: True, "cpu")
    dist.destroy_process_group()
    q.put((rank, out))


def test_peer_memory_handshake_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_handshake_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    expect_blob = _FakeCG(0).record + _FakeCG(1).record  # rank-major
    for r in range(2):
        assert res[r]["bcast"] == b"nccl-id-" + bytes(120)
        assert res[r]["kept"] is True
        assert res[r]["blob"] == expect_blob
        assert res[r]["kept_when_one_fails"] is False
        assert res[r]["kept_when_attach_fails"] is False
