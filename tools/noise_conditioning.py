"""How sensitive is a network's gradient to a small relative error in its conv / FC outputs? Runs the
fp64 oracle twice on the same batch -- once exact, once with every contraction output multiplied by
(1 + eps * N(0,1)) (eps = the 3xTF32 kernels' measured forward error, Reading 43) -- and prints the
per-tensor rel-L2 between the two gradients (DESIGN.md Reading 28).

    python tools/noise_conditioning.py --net alexnet --hw 227 --batch 2 --eps 2e-5
"""
import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "tests"))
import synthdata  # noqa: E402
from netutil import global_rel, rel  # noqa: E402
from oracle import layers as L  # noqa: E402
from oracle import nets  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="alexnet")
    ap.add_argument("--hw", type=int, default=227)
    ap.add_argument("--batch", type=int, default=2)
    ap.add_argument("--eps", type=float, default=2e-5)
    a = ap.parse_args()
    net = nets.alexnet(in_hw=a.hw) if a.net == "alexnet" else nets.resnet50(in_hw=a.hw)
    params = nets.init_params(net, seed=2)
    g = synthdata.rng(4)
    for k in params:
        if k.endswith(".b"):
            params[k] = g.uniform(-0.05, 0.05, params[k].shape).astype(np.float32)
    x = synthdata.images(a.batch, a.hw, a.hw, 3, seed=0)
    t = synthdata.labels(a.batch, 1000, seed=1)
    _, ref, _ = nets.forward_backward(net, params, x, t, rng=(5, 3))
    noise = synthdata.rng(11)
    orig = {n: getattr(L, n) for n in ("conv2d_fwd", "conv2d_dgrad", "conv2d_wgrad", "fc_fwd", "fc_bwd")}

    def noisy(f):
        def g_(*args, **kw):
            out = f(*args, **kw)
            if isinstance(out, tuple):
                return tuple(o * (1 + a.eps * noise.standard_normal(np.shape(o))) for o in out)
            return out * (1 + a.eps * noise.standard_normal(out.shape))
        return g_
    for n, f in orig.items():
        setattr(L, n, noisy(f))
    try:
        _, got, _ = nets.forward_backward(net, params, x, t, rng=(5, 3))
    finally:
        for n, f in orig.items():
            setattr(L, n, f)
    per = sorted(((k, rel(got[k], ref[k])) for k in ref), key=lambda kv: -kv[1])
    print(json.dumps({"net": a.net, "hw": a.hw, "batch": a.batch, "eps": a.eps, "global": global_rel(got, ref),
                      "worst": per[:8]}, indent=1))


if __name__ == "__main__":
    main()
