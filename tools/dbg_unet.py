"""Per-tensor gradient rel-L2 of the 3D U-Net step vs the oracle (debug aid)."""
import sys, os
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synthdata
from oracle import nets
from netutil import global_rel, load_params, pad_input, read_params, rel
import test_gpu_3d as T
E = int(os.environ.get("E", "16")); T.E = E
net = nets.unet3d(in_d=E, width=32, classes=2)
params = nets.init_params(net, seed=21, bn_random=True)
g = synthdata.rng(22)
x = g.standard_normal((1, E, E, E, 1)).astype(np.float32)
t = g.integers(0, 2, (1, E, E, E))
for prec in ("fp64", "tf32"):
    loss, grads, _ = nets.forward_backward(net, params, x, t, precision=prec)
    u = dict(params=params, x=x, t=t)
    ctx = T._ctx(2 << 30, 512 << 20)
    ctx.profile(1)
    l2, _, _ = T._step(ctx, u, "incore")
    gg = read_params(ctx, params, 1)
    print(prec, "loss", loss, l2, "global", global_rel(gg, grads))
    if prec == "fp64":
        for k in grads:
            r = rel(gg[k], grads[k])
            if r > 2e-3: print("  ", k, "%.2e" % r, "norm %.3e" % np.linalg.norm(grads[k]))
    ctx.close()
