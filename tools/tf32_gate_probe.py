"""Probe: with single-TF32 contractions (precision 0, the north_star's "TF32 in, FP32 accumulate"),
how far are the gradients from the fp64 oracle when both sides take the GPU's own ReLU / max-pool
decisions (Reading 28)? Prints per-tensor worst errors for the tiny CNN and ResNet-50 (224^2,
batch 8, standard and small-residual init) at precision 0 and 1. GPU box only."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "tests"))
sys.path.insert(0, os.path.join(HERE, ".."))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthdata  # noqa: E402
from gates import gpu_decisions, step_for_decisions  # noqa: E402
from netutil import global_rel, read_params, rel  # noqa: E402
from oracle import nets  # noqa: E402
import test_gpu_train as T  # noqa: E402


def case(name, init):
    if name == "tiny":
        net = nets.tiny_cnn()
        params = nets.init_params(net, seed=2, bn_random=True)
        x, t = synthdata.images(8, 32, 32, 3, seed=0), synthdata.labels(8, 10, seed=1)
        ctx = T._ctx_for("tiny", 8, 32, 10, 256 << 20, 64 << 20)
    else:
        net = nets.resnet50(in_hw=224, classes=1000)
        params = (nets.init_params(net, seed=2, bn_random=True, residual_gamma=(0.1, 0.3)) if init == "small"
                  else nets.init_params(net, seed=2))
        x, t = synthdata.images(8, 224, 224, 3, seed=0), synthdata.labels(8, 1000, seed=1)
        ctx = T._ctx_for("resnet50", 8, 224, 1000, 4 << 30, 2 << 30)
    ctx.profile(1)
    return net, params, x, t, ctx


for name, init in (("tiny", ""), ("r50", "small"), ("r50", "standard")):
    net, params, x, t, ctx = case(name, init)
    for prec in (1, 0):
        ctx.set_precision(prec)
        ctx.profile(1)
        step_for_decisions(ctx, lambda: T._step(ctx, params, x, t, "incore"))
        dec = gpu_decisions(ctx, net)
        g = read_params(ctx, params, 1)
        _, ref, _ = nets.forward_backward(net, params, x, t, decisions=dec)
        rows = sorted(((k, rel(g[k], ref[k])) for k in ref if np.linalg.norm(ref[k]) > 0), key=lambda r: -r[1])
        w = [r for r in rows if r[0].endswith(".w")]
        print("%-4s %-8s prec %d: whole %.2e  worst %s  worst weight %s" % (
            name, init, prec, global_rel(g, ref), "%s %.2e" % rows[0], "%s %.2e" % w[0]), flush=True)
    ctx.close()
