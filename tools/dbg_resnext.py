"""Debug: per-tensor gradient error of the ResNeXt-50 (3D) step against the oracle (GPU)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import test_gpu_resnext3d as T
from netutil import read_params, rel
from oracle import nets
import synthdata

net = nets.resnext3d(T.DHW, classes=T.CLASSES, depth=50)
params = nets.init_params(net, seed=31, bn_random=True)
x = synthdata.rng(32).standard_normal((1,) + T.DHW + (3,)).astype(np.float32)
t = np.array([3])
mg = []
loss, grads, outs = nets.forward_backward(net, params, x, t, map_grads=mg)
_, grads32, _ = nets.forward_backward(net, params, x, t, precision="fp32")
os.environ["POOCH_DEBUG_NO_REUSE"] = "1"
ctx = T._ctx(2 << 30, 64 << 20)
ctx.profile(1)
l2, _, _ = T._step(ctx, dict(params=params, x=x, t=t), "incore")
print("loss", loss, l2)
g = read_params(ctx, params, 1)
for k in nets.param_shapes(net):
    print("%-32s %.3e  fp32-oracle %.3e" % (k, rel(g[k], grads[k]), rel(grads32[k], grads[k])))
# forward maps and map gradients (in-core plan: every instance live)
for i, tk in enumerate(net.tasks):
    shp = outs[i].shape
    nb = int(np.prod(shp)) * 4
    if tk.kind == "fc_ce":
        continue
    m = ctx.read_buffer(0, i, nb)
    ref = np.moveaxis(outs[i], 1, -1).reshape(-1)
    gm = ctx.read_buffer(2, i, nb)
    gref = np.moveaxis(mg[i], 1, -1).reshape(-1) if mg[i] is not None else None
    print("%3d %-26s %-10s map %.2e  grad %s" % (i, tk.name, tk.kind, rel(m, ref),
          "%.2e" % rel(gm, gref) if gref is not None else "-"))
