import sys, numpy as np, torch
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import synthdata
from oracle import nets
from netutil import load_params, pad_input, read_params, rel
from test_gpu_train import _ctx_for, _put_batch
net = nets.tiny_cnn(); params = nets.init_params(net, seed=2, bn_random=True)
x = synthdata.images(8, 32, 32, 3, seed=0); t = synthdata.labels(8, 10, seed=1)
loss, grads, outs = nets.forward_backward(net, params, x, t)
ctx = _ctx_for("tiny", 8, 32, 10, 256 << 20, 64 << 20)
ctx.profile(1)
load_params(ctx, params); _put_batch(ctx, x, t)
ctx.plan("incore")
l = ctx.train_step(0.0)
print("loss", l, loss)
for i, tk in enumerate(net.tasks):
    c, h, w = tk.out_chw
    ref = outs[i]
    if ref.ndim == 4:
        ref = ref.transpose(0, 2, 3, 1)
    ref = ref.reshape(8, -1)
    cp = c if tk.kind != 'fc_ce' else 12
    got = ctx.read_buffer(0, i, 8 * cp * h * w * 4).reshape(8, h, w, cp)[..., :c].reshape(8, -1)
    print(i, tk.name, tk.kind, "rel", rel(got, ref), "nan", np.isnan(got).sum(), got.ravel()[:4], ref.ravel()[:4])
g = read_params(ctx, params, 1)
for k in g: print(k, rel(g[k], grads[k]))
