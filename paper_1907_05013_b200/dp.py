"""Data-parallel plumbing (host side): ranks agree on one plan.

Every rank runs its own out-of-core executor on its own mini-batch shard
(weak scaling, BASELINE.json config 5); the only exchange inside the step is
the NCCL gradient allreduce done by libpooch.so. Before planning, the ranks
take the element-wise maximum of their measured profiles (DESIGN.md Reading
29) so that every rank plans -- deterministically -- the same classification
and its swap traffic is sized for the slowest rank.
"""
from __future__ import annotations

KEYS = ("fwd", "bwd", "rec", "d2h", "h2d")


def agree_profile(prof: dict, group=None, device="cpu") -> dict:
    """Element-wise max of every rank's profile (torch.distributed all_reduce MAX)."""
    import torch
    import torch.distributed as dist
    n = len(prof["fwd"])
    t = torch.tensor([list(prof[k]) for k in KEYS] + [[int(prof["tail"])] * n], dtype=torch.int64,
                     device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    a = t.cpu().tolist()
    out = dict(prof)
    for i, k in enumerate(KEYS):
        out[k] = a[i]
    out["tail"] = a[len(KEYS)][0]
    return out


def broadcast_unique_id(rank: int, group=None, device="cpu") -> bytes:
    """Rank 0 creates the 128-byte ncclUniqueId (libnccl, loaded by torch); all ranks get it."""
    import ctypes

    import torch
    import torch.distributed as dist
    buf = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        lib = ctypes.CDLL("libnccl.so.2")
        raw = ctypes.create_string_buffer(128)
        if lib.ncclGetUniqueId(raw) != 0:
            raise RuntimeError("ncclGetUniqueId failed")
        buf.copy_(torch.frombuffer(bytearray(raw.raw), dtype=torch.uint8))
    dist.broadcast(buf, 0, group=group)
    return bytes(buf.cpu().numpy().tobytes())
