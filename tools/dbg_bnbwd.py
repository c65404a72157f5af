import sys, os, numpy as np, torch
os.environ["POOCH_DEBUG_NO_REUSE"] = "1"
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import synthdata
from oracle import nets, layers as L
from netutil import load_params, pad_input, read_params, rel
from test_gpu_train import _ctx_for, _put_batch
net = nets.tiny_cnn(); B = 8
ctx = _ctx_for("tiny", B, 32, 10, 256 << 20, 64 << 20)
params = nets.init_params(net, seed=2, bn_random=True)
x = synthdata.images(B, 32, 32, 3, seed=0); t = synthdata.labels(B, 10, seed=1)
ctx.profile(1); load_params(ctx, params); _put_batch(ctx, x, t); ctx.plan("incore"); ctx.train_step(0.0)
def rd(w, m): return ctx.read_buffer(w, m, B*32*32*32*4).reshape(B,32,32,32).transpose(0,3,1,2).astype(np.float64)
c = rd(0, 4); gy = rd(2, 5); gc_gpu = rd(2, 4)
gam = params["bn2.gamma"].astype(np.float64); bet = params["bn2.beta"].astype(np.float64)
y, cache = L.bn_fwd(c, gam, bet)
dz = L.relu_bwd(gy, np.maximum(y, 0))
dx, dg, db = L.bn_bwd(dz, cache, gam)
print("g(conv2) rel", rel(gc_gpu, dx))
g = read_params(ctx, params, 1)
print("dgamma rel", rel(g["bn2.gamma"], dg), "dbeta rel", rel(g["bn2.beta"], db))
print("cancellation |sum dz| / sum|dz| per channel (median)", np.median(np.abs(dz.sum((0,2,3))) / np.abs(dz).sum((0,2,3))))
print("dbeta gpu", g["bn2.beta"][:6]); print("dbeta ref", db[:6])
