"""Per-shape conv pass timings over every ResNet-50 v1.5 conv (fwd / dgrad / wgrad), weighted by
how often the shape occurs, against each pass's roofline time max(flops / P_tensor, bytes / BW).

Usage (GPU box): B=256 PREC=1 python tools/kbench_r50.py  -> gpurun_out/kbench_r50_B{B}.json
"""
import ctypes as C
import collections
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from oracle import nets  # noqa: E402  (layer shapes only)
from paper_1907_05013_b200 import _lib  # noqa: E402

B = int(os.environ.get("B", "256"))
PREC = int(os.environ.get("PREC", "1"))
pk = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
BW = pk.get("hbm_gbs", 6550.0) * 1e9
PT = pk.get("bf16_tflops_sustained", 1368.0) * 1.1 / 2.25 / (3 if PREC else 1) * 1e12

net = nets.resnet50()
shapes = collections.Counter()
first = {}
for i, t in enumerate(net.tasks):
    if t.kind != "conv":
        continue
    cin = 4 if t.inputs[0] < 0 else t.cin
    src = net.tasks[t.inputs[0]] if t.inputs[0] >= 0 else None
    H = src.out_chw[1] if src is not None else 224
    key = (H, cin, t.out_chw[0], t.k, t.stride, t.pad)
    shapes[key] += 1
    first.setdefault(key, t.name)

res = []
tot_meas = tot_roof = 0.0
for key, cnt in shapes.items():
    H, Cin, K, R, s, p = key
    Ho = (H + 2 * p - R) // s + 1
    x = torch.randn(B, H, H, Cin, device="cuda")
    w = torch.randn(K, R, R, Cin, device="cuda") * 0.05
    y = torch.empty(B, Ho, Ho, K, device="cuda")
    gy = torch.randn(B, Ho, Ho, K, device="cuda")
    wt = w.permute(3, 1, 2, 0).contiguous()
    dx = torch.empty_like(x)
    dw = torch.empty_like(w)
    d = _lib.ConvDesc(B, H, H, Cin, K, R, R, s, p, PREC)
    mt = _lib.lib.pooch_op_conv_stat_tiles(C.byref(d))
    s1 = torch.empty(mt, K, device="cuda")
    s2 = torch.empty(mt, K, device="cuda")
    wsb = _lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d))
    ws = torch.empty(max(wsb // 4, 1), device="cuda")
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    ops = {
        "fwd": lambda: _lib.lib.pooch_op_conv_fwd(C.byref(d), P(x), P(w), P(y), P(s1), P(s2), None),
        "dgrad": lambda: _lib.lib.pooch_op_conv_dgrad(C.byref(d), P(gy), P(wt), P(dx), 0, None),
        "wgrad": lambda: _lib.lib.pooch_op_conv_wgrad(C.byref(d), P(x), P(gy), P(dw), P(ws), wsb, None),
    }
    flops = 2.0 * B * Ho * Ho * K * R * R * Cin
    byt = 4.0 * (x.numel() + gy.numel() + w.numel())
    roof_ms = max(flops / PT, byt / BW) * 1e3
    for op, f in ops.items():
        if H == 224 and op == "dgrad":
            continue
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        r = dict(layer=first[key], shape=list(key), count=cnt, op=op, ms=round(ms, 4), roof_ms=round(roof_ms, 4),
                 frac=round(roof_ms / ms, 3), tflops=round(flops / ms / 1e9, 1), gap_ms_total=round((ms - roof_ms) * cnt, 3))
        tot_meas += ms * cnt
        tot_roof += roof_ms * cnt
        res.append(r)
        print(json.dumps(r), flush=True)
res.sort(key=lambda r: -r["gap_ms_total"])
print("total conv time %.2f ms, roofline %.2f ms (frac %.3f)" % (tot_meas, tot_roof, tot_roof / tot_meas))
for r in res[:15]:
    print("%-22s %-6s x%-2d %7.3f ms roof %7.3f frac %.2f gap %.2f ms" % (r["layer"], r["op"], r["count"], r["ms"],
                                                                        r["roof_ms"], r["frac"], r["gap_ms_total"]))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(dict(batch=B, prec=PREC, total_ms=tot_meas, roof_ms=tot_roof, rows=res),
          open("gpurun_out/kbench_r50_B%d.json" % B, "w"), indent=1)
