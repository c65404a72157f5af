"""One rank of the multi-process peer-allreduce test (tests/test_gpu_peer.py); not a test module.

Every rank runs on cuda:0 (the GPU boxes have one GPU; the exchange buffers are then mapped
between processes of the same device, the same cudaIpc path as NVLink peers). Each rank:
  1. steps a context WITHOUT exchange on its own shard -> its local gradient g_r;
  2. steps a context WITH the peer-memory allreduce (pooch_peer_open / pooch_set_peers) on the
     same shard, same parameters, under the plan `strategy`, twice (graph capture + replay);
  3. writes its gradients / parameters / loss to <out>/rank<r>.npz.
The test checks that every rank's exchanged gradient equals sum_r g_r formed in rank order in
fp32, bit for bit, and that the parameters after the update agree across ranks.
argv: out_dir strategy net
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synthdata  # noqa: E402
from netutil import load_params, pad_input  # noqa: E402
from oracle import nets  # noqa: E402

LR = 0.05


def main():
    out, strategy, netname = sys.argv[1], sys.argv[2], sys.argv[3]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%s" % os.environ["MASTER_PORT"], rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    from paper_1907_05013_b200 import dp
    from paper_1907_05013_b200.executor import Context

    if netname == "tiny":
        model, batch, hw, classes, dev_b = nets.tiny_cnn(), 8, 32, 10, 256 << 20
    else:
        model, batch, hw, classes, dev_b = nets.resnet50(in_hw=64, classes=100), 4, 64, 100, 2 << 30
    params = nets.init_params(model, seed=2, bn_random=True)
    x = synthdata.images(batch, hw, hw, 3, seed=100 + rank)
    t = synthdata.labels(batch, classes, seed=200 + rank)

    def make_ctx(peers):
        ctx = Context.builtin(netname, batch, in_hw=hw, classes=classes)
        dev = torch.empty(dev_b, dtype=torch.uint8, device="cuda")
        host = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
        ctx.set_budget(dev, dev_b, host, host.numel())
        ss = [torch.cuda.Stream() for _ in range(4)]
        ctx.set_streams(*ss)
        ctx._torch = (dev, host, ss)
        if peers:
            dp.setup_peers(ctx, rank, world)
        xp, lp = ctx.input_slot()
        base = dev.data_ptr()
        xt = torch.from_numpy(pad_input(x)).reshape(-1).cuda()
        lt = torch.from_numpy(t.astype(np.int32)).cuda()
        dev[xp - base: xp - base + xt.numel() * 4].view(torch.float32).copy_(xt)
        dev[lp - base: lp - base + lt.numel() * 4].view(torch.int32).copy_(lt)
        torch.cuda.synchronize()
        return ctx

    def grads(ctx):
        return [ctx.get_param(i, 1).copy() for i in range(len(ctx.params()))]

    def weights(ctx):
        return [ctx.get_param(i, 0).copy() for i in range(len(ctx.params()))]

    # 1. local gradient (no exchange, world 1)
    c0 = make_ctx(False)
    c0.profile(1)
    load_params(c0, params)
    c0.plan("incore")
    loss_local = c0.train_step(LR)
    torch.cuda.synchronize()
    g_local = grads(c0)
    c0.close()

    # 2. exchanged, under the plan `strategy`: two steps from the same state (capture, replay)
    c1 = make_ctx(True)
    nr, rk, _ = c1.comm_info()
    c1.profile(1)
    res = {}
    for it in range(2):
        load_params(c1, params)
        if it == 0:
            cls, _ = c1.plan(strategy)
        loss = c1.train_step(LR)
        torch.cuda.synchronize()
        res["loss%d" % it] = float(loss)
        res["graph%d" % it] = bool(c1.step_was_graph())
        g = grads(c1)
        w = weights(c1)
        np.savez(os.path.join(out, "rank%d_it%d.npz" % (rank, it)), *g)
        np.savez(os.path.join(out, "rank%d_w%d.npz" % (rank, it)), *w)
    np.savez(os.path.join(out, "rank%d_local.npz" % rank), *g_local)
    res.update(rank=rank, world=world, comm_nranks=nr, comm_rank=rk, loss_local=float(loss_local),
               plan=[int(v) for v in cls], peer_bytes=int(c1.peer_bytes))
    with open(os.path.join(out, "rank%d.json" % rank), "w") as f:
        json.dump(res, f)
    c1.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
