"""3D U-Net gradient gate vs parameter init (ReLU / max-pool decision sensitivity)."""
import sys, os
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synthdata
from oracle import nets
from netutil import global_rel, read_params, rel
import test_gpu_3d as T
for E, shift, gscale in ((16, 0.0, 1.0), (16, 1.0, 1.0), (16, 1.0, 0.5), (16, 2.0, 0.5), (32, 0.0, 1.0), (32, 1.0, 0.5)):
    T.E = E
    net = nets.unet3d(in_d=E, width=32, classes=2)
    params = nets.init_params(net, seed=21, bn_random=True)
    for k in params:
        if k.endswith(".beta"): params[k] = (params[k] + shift).astype(np.float32)
        if k.endswith(".gamma"): params[k] = (params[k] * gscale).astype(np.float32)
    g = synthdata.rng(22)
    x = g.standard_normal((1, E, E, E, 1)).astype(np.float32)
    t = g.integers(0, 2, (1, E, E, E))
    loss, grads, _ = nets.forward_backward(net, params, x, t)
    u = dict(params=params, x=x, t=t)
    ctx = T._ctx(2 << 30, 512 << 20)
    ctx.profile(1)
    l2, _, _ = T._step(ctx, u, "incore")
    gg = read_params(ctx, params, 1)
    worst = max((rel(gg[k], grads[k]), k) for k in grads if np.linalg.norm(grads[k]) > 0)
    print("E", E, "beta+", shift, "gamma*", gscale, "loss %.7f %.7f" % (loss, l2), "global %.2e" % global_rel(gg, grads), "worst %.2e %s" % worst, flush=True)
    ctx.close()
