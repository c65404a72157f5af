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
    # host-link rates (Reading 51): the most pessimistic duplex factor, the same on every rank
    if "duplex_gbs" in prof:
        r = torch.tensor([-float(prof["duplex_gbs"]), float(prof["d2h_gbs"]), float(prof["h2d_gbs"])],
                         dtype=torch.float64, device=device)
        dist.all_reduce(r, op=dist.ReduceOp.MAX, group=group)
        out["duplex_gbs"], out["d2h_gbs"], out["h2d_gbs"] = -float(r[0]), float(r[1]), float(r[2])
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


def setup_peers(ctx, rank: int, world: int, group=None):
    """Peer-memory allreduce (libpooch's own, peer.cu): each rank exports its exchange buffer,
    the 64-byte IPC handles are all-gathered over the (gloo / nccl) process group, every rank
    maps every other rank's buffer. Returns the exchange buffer's bytes (outside the arena)."""
    import torch.distributed as dist
    h = ctx.peer_open(rank, world)
    handles = [None] * world
    if world > 1:
        dist.all_gather_object(handles, h, group=group)
    else:
        handles = [h]
    ctx.set_peers(handles)
    return ctx.peer_bytes


def relaunch_argv(script: str, argv, nproc: int, port: int):
    """`bench.py --gpus N` run without a launcher (WORLD_SIZE unset) re-executes itself under
    torch.distributed.run with one process per GPU on 127.0.0.1 -- the driver's own launch line."""
    import sys
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % nproc,
            "--master-addr", "127.0.0.1", "--master-port", str(port), script] + list(argv)


def pci_numa_node(bus_id: str) -> int:
    """NUMA node of a PCI device from sysfs (-1 when unknown / single-node)."""
    bus_id = bus_id.lower()
    if bus_id.count(":") == 1:
        bus_id = "0000:" + bus_id
    try:
        with open("/sys/bus/pci/devices/%s/numa_node" % bus_id) as f:
            return int(f.read().strip())
    except (OSError, ValueError):
        return -1


def node_cpus(node: int):
    """CPU ids of a NUMA node (sysfs cpulist, e.g. '0-15,32-47')."""
    try:
        with open("/sys/devices/system/node/node%d/cpulist" % node) as f:
            spec = f.read().strip()
    except OSError:
        return []
    out = []
    for part in spec.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


def bind_host_to_gpu(device: int) -> int:
    """Pin this rank's CPU affinity to its GPU's NUMA node, so that the pinned host arena it
    registers next (first touch by this thread) lands in that node's memory and the swap copies
    cross no inter-socket link. Returns the node, or -1 when the box has no NUMA information."""
    import os

    import torch
    p = torch.cuda.get_device_properties(device)
    bus = getattr(p, "pci_bus_id", None)
    if bus is None:
        return -1
    bus_id = "%04x:%02x:%02x.0" % (getattr(p, "pci_domain_id", 0), bus, getattr(p, "pci_device_id", 0))
    node = pci_numa_node(bus_id)
    cpus = node_cpus(node) if node >= 0 else []
    allowed = os.sched_getaffinity(0)
    cpus = [c for c in cpus if c in allowed]
    if cpus:
        os.sched_setaffinity(0, cpus)
    return node if cpus else -1


def digest(arrays) -> str:
    """sha256 over the bytes of a list of arrays (parameter checksum for rank consistency)."""
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(memoryview(a).cast("B"))
    return h.hexdigest()


def ranks_identical(local_digest: str, group=None) -> bool:
    """True when every rank holds the same digest (all_gather_object)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return True
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, local_digest, group=group)
    return all(d == out[0] for d in out)
