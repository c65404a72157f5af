"""Micro-benchmark of the conv passes on ResNet-50 layer shapes (CUDA events)."""
import ctypes as C, sys, os, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1907_05013_b200 import _lib
B = int(os.environ.get("B", "256"))
PREC = int(os.environ.get("PREC", "1"))
shapes = [  # name, H, C, K, R, stride
    ("stem7x7", 224, 4, 64, 7, 2), ("l1.c1 1x1", 56, 256, 64, 1, 1), ("l1.c2 3x3", 56, 64, 64, 3, 1),
    ("l1.c3 1x1", 56, 64, 256, 1, 1), ("l2.c2 3x3", 28, 128, 128, 3, 1), ("l3.c2 3x3", 14, 256, 256, 3, 1),
    ("l3.c3 1x1", 14, 256, 1024, 1, 1), ("l4.c2 3x3", 7, 512, 512, 3, 1), ("l4.c1 1x1", 7, 2048, 512, 1, 1),
    ("l2.c2s2 3x3", 56, 128, 128, 3, 2), ("l2.ds 1x1s2", 56, 256, 512, 1, 2)]
OPS = os.environ.get("OPS", "fwd,dgrad,wgrad").split(",")
only = os.environ.get("ONLY")
res = []
for name, H, Cin, K, R, s in shapes:
    if only and only not in name: continue
    p = R // 2
    Ho = (H + 2 * p - R) // s + 1
    x = torch.randn(B, H, H, Cin, device="cuda"); w = torch.randn(K, R, R, Cin, device="cuda") * 0.05
    y = torch.empty(B, Ho, Ho, K, device="cuda"); gy = torch.randn(B, Ho, Ho, K, device="cuda")
    wt = w.permute(3, 1, 2, 0).contiguous(); dx = torch.empty_like(x); dw = torch.empty_like(w)
    d = _lib.ConvDesc(B, H, H, Cin, K, R, R, s, p, PREC)
    mt = _lib.lib.pooch_op_conv_stat_tiles(C.byref(d))
    s1 = torch.empty(mt, K, device="cuda"); s2 = torch.empty(mt, K, device="cuda")
    wsb = _lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d)); ws = torch.empty(max(wsb // 4, 1), device="cuda")
    P = lambda t: C.c_void_p(t.data_ptr())
    ops = {
        "fwd": lambda: _lib.lib.pooch_op_conv_fwd(C.byref(d), P(x), P(w), P(y), P(s1), P(s2), None),
        "dgrad": lambda: _lib.lib.pooch_op_conv_dgrad(C.byref(d), P(gy), P(wt), P(dx), 0, None),
        "wgrad": lambda: _lib.lib.pooch_op_conv_wgrad(C.byref(d), P(x), P(gy), P(dw), P(ws), wsb, None),
    }
    flops = 2.0 * B * Ho * Ho * K * R * R * Cin
    for op, f in ops.items():
        if (name.startswith("stem") and op == "dgrad") or op not in OPS: continue
        for _ in range(2): f()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        n = 5
        e0.record()
        for _ in range(n): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        byt = 4.0 * (x.numel() + gy.numel() + w.numel())
        r = dict(layer=name, op=op, ms=round(ms, 3), tflops=round(flops / ms / 1e9, 1), gbs=round(byt / ms / 1e6, 1))
        res.append(r); print(r, flush=True)
json.dump(res, open("gpurun_out/kbench_B%d_P%d.json" % (B, PREC), "w"), indent=1)
