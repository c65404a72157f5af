"""Per-map forward rel-L2 of the 3D U-Net (in-core) vs the oracle -- finds the first layer that drifts."""
import sys, os
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synthdata
from oracle import nets
from netutil import rel
import test_gpu_3d as T
E = int(os.environ.get("E", "16")); T.E = E
net = nets.unet3d(in_d=E, width=32, classes=2)
params = nets.init_params(net, seed=21, bn_random=True)
g = synthdata.rng(22)
x = g.standard_normal((1, E, E, E, 1)).astype(np.float32)
t = g.integers(0, 2, (1, E, E, E))
mg = []
loss, grads, outs = nets.forward_backward(net, params, x, t, map_grads=mg)
u = dict(params=params, x=x, t=t)
ctx = T._ctx(2 << 30, 512 << 20)
ctx.profile(1)
l2, _, _ = T._step(ctx, u, "incore")
print("loss", loss, l2)
for m, task in enumerate(net.tasks):
    ref = np.moveaxis(outs[m], 1, -1)
    nb = ref.size * 4
    if task.kind == "head_ce":
        nb = ref.size // ref.shape[-1] * 4 * 4
        got = ctx.read_buffer(0, m, nb).reshape(ref.shape[:-1] + (4,))[..., :ref.shape[-1]]
    else:
        got = ctx.read_buffer(0, m, nb).reshape(ref.shape)
    gr = ""
    if mg[m] is not None and m < len(net.tasks) - 1:
        gref = np.moveaxis(mg[m], 1, -1)
        ggot = ctx.read_buffer(2, m, gref.size * 4).reshape(gref.shape)
        gr = "grad %.2e" % rel(ggot, gref)
    print("%-12s %-8s fwd %.2e %s" % (task.name, task.kind, rel(got, ref), gr))
