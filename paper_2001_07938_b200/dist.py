"""Host-side plumbing of the sharded CG driver across processes
(torch.distributed): the NCCL unique id broadcast and the peer-memory
handshake (each rank's 208-byte record — CUDA IPC handles and column
footprint — all-gathered rank-major, then kept only if every rank agrees)."""
from __future__ import annotations

import sys


def broadcast_bytes(payload: bytes | None, nbytes: int, device) -> bytes:
    """Rank 0's `payload` (nbytes) on every rank."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if dist.get_rank() == 0:
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tobytes())


def all_gather_records(record: bytes, device) -> bytes:
    """Every rank's fixed-size record, concatenated in rank order."""
    import torch
    import torch.distributed as dist
    mine = torch.frombuffer(bytearray(record), dtype=torch.uint8).to(device)
    out = [torch.empty_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(out, mine)
    return b"".join(bytes(o.cpu().numpy().tobytes()) for o in out)


def all_agree(ok: bool, device) -> bool:
    """True on every rank iff `ok` on every rank."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([1.0 if ok else 0.0], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item() == 1.0)


def attach_peer_memory(cg, verify, device) -> bool:
    """Switch a DistCG (NCCL driver) to the peer-memory exchange; `verify()`
    runs the sharded benchmark and says whether it verified. Returns whether
    every rank kept it (False: the caller recreates the NCCL driver)."""
    import torch.distributed as dist
    try:
        cg.p2p_attach(all_gather_records(cg.p2p_export(), device))
        ok = bool(verify())
    except Exception as e:  # noqa: BLE001 - any failure falls back to NCCL
        print(f"rank {dist.get_rank()}: peer-memory exchange unavailable ({e}); using NCCL", file=sys.stderr)
        ok = False
    return all_agree(ok, device)
