import sys, os, numpy as np, torch
os.environ["POOCH_DEBUG_NO_REUSE"] = "1"
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import synthdata
from oracle import nets
from netutil import load_params, pad_input, read_params, rel
from test_gpu_train import _ctx_for, _put_batch
net = nets.tiny_cnn(); params = nets.init_params(net, seed=2, bn_random=True)
x = synthdata.images(8, 32, 32, 3, seed=0); t = synthdata.labels(8, 10, seed=1)
gm = []
loss, grads, outs = nets.forward_backward(net, params, x, t, map_grads=gm)
ctx = _ctx_for("tiny", 8, 32, 10, 256 << 20, 64 << 20)
ctx.profile(1)
load_params(ctx, params); _put_batch(ctx, x, t)
ctx.plan("incore")
l = ctx.train_step(0.0)
print("loss", l, loss)
for i, tk in enumerate(net.tasks):
    c, h, w = tk.out_chw
    cp = c if tk.kind != 'fc_ce' else 12
    for which, ref in ((0, outs[i]), (2, gm[i])):
        if ref is None: continue
        ref = ref.transpose(0, 2, 3, 1).reshape(8, -1) if ref.ndim == 4 else ref.reshape(8, -1)
        got = ctx.read_buffer(which, i, 8 * cp * h * w * 4).reshape(8, h, w, cp)[..., :c].reshape(8, -1)
        print(i, tk.name, "map" if which == 0 else "grad", "rel %.3g" % rel(got, ref), got.ravel()[:3], ref.ravel()[:3])
g = read_params(ctx, params, 1)
for k in g: print(k, rel(g[k], grads[k]))
