"""3D U-Net: isolate BN-backward error with the GPU's own inputs (no region reuse)."""
import sys, os
os.environ["POOCH_DEBUG_NO_REUSE"] = "1"
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synthdata
from oracle import nets, layers as L
from netutil import rel, read_params
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
def rd(which, m):
    ref = np.moveaxis(outs[m], 1, -1)
    return ctx.read_buffer(which, m, ref.size * 4).reshape(ref.shape).astype(np.float64)
for m, task in enumerate(net.tasks[:-1]):
    ref = np.moveaxis(outs[m], 1, -1)
    gref = np.moveaxis(mg[m], 1, -1) if mg[m] is not None else None
    s = "%-12s fwd %.2e" % (task.name, rel(rd(0, m), ref))
    if gref is not None: s += " grad %.2e" % rel(rd(2, m), gref)
    if task.kind == "bnrelu":   # BN bwd with the GPU's own inputs, fp64
        c = np.moveaxis(rd(0, task.inputs[0]), -1, 1); gy = np.moveaxis(rd(2, m), -1, 1)
        gam = params[task.name + ".gamma"].astype(np.float64); bet = params[task.name + ".beta"].astype(np.float64)
        yb, cache = L.bn_fwd(c, gam, bet)
        dz = L.relu_bwd(gy, np.maximum(yb, 0))
        dx, dg, db = L.bn_bwd(dz, cache, gam)
        s += "  | bn-bwd kernel vs fp64(GPU inputs): %.2e" % rel(np.moveaxis(rd(2, task.inputs[0]), -1, 1), dx)
    print(s)
