"""Probe: can two NCCL ranks share one GPU on this image (NCCL 2.28)? Prints the outcome.
Run: python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/nccl_same_gpu_probe.py"""
import os
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
try:
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    t = torch.full((4,), float(rank + 1), device="cuda")
    dist.all_reduce(t)
    torch.cuda.synchronize()
    print("rank", rank, "allreduce ok", t.tolist(), flush=True)
    dist.destroy_process_group()
except Exception as e:
    print("rank", rank, "FAILED:", type(e).__name__, str(e)[:300], flush=True)
