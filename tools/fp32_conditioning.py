"""How far does plain fp32 arithmetic alone move ResNet-50 gradients from fp64? Runs the oracle
twice on the same seeded batch -- fp64 and its fp32 mode (the same NumPy code in float32) -- and
prints the whole-gradient and per-tensor rel-L2, per parameter family (DESIGN.md Reading 28).

    python tools/fp32_conditioning.py [--batch 8] [--hw 224] [--init standard|test] [--out f.json]
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
from oracle import nets  # noqa: E402


def family(k):
    if k.endswith(".w") or k.endswith(".b"):
        return "fc" if k.startswith("fc") else "conv"
    return "bn"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--hw", type=int, default=224)
    ap.add_argument("--init", default="standard", choices=["standard", "test"])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    net = nets.resnet50(in_hw=a.hw, classes=1000)
    if a.init == "standard":
        params = nets.init_params(net, seed=2)
    else:
        params = nets.init_params(net, seed=2, bn_random=True, residual_gamma=(0.1, 0.3))
    x = synthdata.images(a.batch, a.hw, a.hw, 3, seed=0)
    t = synthdata.labels(a.batch, 1000, seed=1)
    l64, g64, _ = nets.forward_backward(net, params, x, t)
    l32, g32, _ = nets.forward_backward(net, params, x, t, precision="fp32")
    per = {k: rel(g32[k], g64[k]) for k in g64}
    fam = {}
    for k, v in per.items():
        fam.setdefault(family(k), []).append(v)
    res = {"batch": a.batch, "hw": a.hw, "init": a.init, "loss64": float(l64), "loss32": float(l32),
           "global_rel": global_rel(g32, g64),
           "family_max": {f: max(v) for f, v in fam.items()},
           "family_median": {f: float(np.median(v)) for f, v in fam.items()},
           "worst": sorted(per.items(), key=lambda kv: -kv[1])[:10]}
    print(json.dumps(res, indent=1))
    if a.out:
        json.dump({"summary": res, "per_tensor": per}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
