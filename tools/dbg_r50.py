import sys, os, numpy as np, torch
os.environ["POOCH_DEBUG_NO_REUSE"] = "1"
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import synthdata
from oracle import nets
from netutil import load_params, pad_input, read_params, rel
from test_gpu_train import _ctx_for, _put_batch
which = sys.argv[1] if len(sys.argv) > 1 else "r50"
if which == "r50":
    hw = int(os.environ.get("HW", "64")); B = int(os.environ.get("B", "4")); ncls = int(os.environ.get("NCLS", "100"))
    net = nets.resnet50(in_hw=hw, classes=ncls)
    ctx = _ctx_for("resnet50", B, hw, ncls, 4 << 30, 2 << 30)
else:
    net = nets.tiny_cnn(); B = 8; hw = 32; ncls = 10
    ctx = _ctx_for("tiny", B, hw, ncls, 256 << 20, 64 << 20)
init = os.environ.get("INIT", "random")
params = nets.init_params(net, seed=2, bn_random=(init != "bench"))
if init == "smallres":
    g0 = np.random.default_rng(9)
    for k in params:
        if k.endswith(".gamma3"):
            params[k] = g0.uniform(0.1, 0.3, params[k].shape).astype(np.float32)
x = synthdata.images(B, hw, hw, 3, seed=0); t = synthdata.labels(B, ncls, seed=1)
gm = []
loss, grads, outs = nets.forward_backward(net, params, x, t, map_grads=gm, precision=os.environ.get("ORACLE_PREC", "fp64"))
ctx.profile(1)
load_params(ctx, params); _put_batch(ctx, x, t)
ctx.plan("incore")
l = ctx.train_step(0.0)
print("loss", l, loss)
from netutil import global_rel
g_all = read_params(ctx, params, 1)
print("INIT", init, "global rel-L2 %.3e" % global_rel(g_all, grads))
if os.environ.get("SHORT"):
    sys.exit(0)
for i in reversed(range(len(net.tasks))):
    tk = net.tasks[i]
    c, h, w = tk.out_chw
    cp = c if tk.kind != 'fc_ce' else (c + 3) // 4 * 4
    s = "%3d %-22s %-9s" % (i, tk.name, tk.kind)
    for which_, ref in ((0, outs[i]), (2, gm[i])):
        if ref is None: s += " grad ---"; continue
        ref = ref.transpose(0, 2, 3, 1).reshape(B, -1) if ref.ndim == 4 else ref.reshape(B, -1)
        got = ctx.read_buffer(which_, i, B * cp * h * w * 4).reshape(B, h, w, cp)[..., :c].reshape(B, -1)
        s += (" map %.2e" if which_ == 0 else " grad %.2e") % rel(got, ref)
    print(s, flush=True)
g = read_params(ctx, params, 1)
errs = sorted(((rel(g[k], grads[k]), k) for k in g), reverse=True)
for e, k in errs[:12]: print("%.3e %s" % (e, k))
if which != "r50":
    # max-pool decision agreement on the pool input (task 7), GPU fp32 values vs oracle fp64
    y_gpu = ctx.read_buffer(0, 7, B * 32 * 32 * 32 * 4).reshape(B, 32, 32, 32)
    y_ora = outs[7].transpose(0, 2, 3, 1)
    def arg(y):
        w = y.reshape(B, 16, 2, 16, 2, 32).transpose(0, 1, 3, 5, 2, 4).reshape(B, 16, 16, 32, 4)
        return np.argmax(w, axis=-1), np.sort(w, axis=-1)
    ag, sg = arg(y_gpu); ao, so = arg(y_ora)
    d = ag != ao
    print("maxpool argmax disagreements", int(d.sum()), "of", d.size)
    print("gap top2 (oracle) at disagreements", (so[..., -1] - so[..., -2])[d][:10])
    print("values gpu", sg[d][:3], "ora", so[d][:3])
    gy = ctx.read_buffer(2, 7, B * 32 * 32 * 32 * 4).reshape(B, 32, 32, 32)
    go = gm[7].transpose(0, 2, 3, 1)
    diff = np.abs(gy - go)
    idx = np.argsort(diff.ravel())[-5:]
    print("largest grad diffs", diff.ravel()[idx], "gpu", gy.ravel()[idx], "ora", go.ravel()[idx])
    print("y at those", y_gpu.ravel()[idx], y_ora.ravel()[idx])
