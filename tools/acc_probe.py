"""Accuracy / speed of the wgrad split length (tensor-core accumulation bias, DESIGN Reading 28).

For a few ResNet-50 / tiny-CNN wgrad shapes: rel-L2 of dW against fp64 (numpy) and the kernel time,
for POOCH_WGRAD_KMAX = 0 (cost-model splits only) and a few caps. GPU box:
    python tools/acc_probe.py > gpurun_out/acc_probe.log
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import layers as L  # noqa: E402
from paper_1907_05013_b200 import _lib  # noqa: E402

P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
shapes = [("tiny conv", 8, 32, 32, 32, 3, 1, 1), ("l1.c2 b8", 8, 56, 64, 64, 3, 1, 1),
          ("l1.c3 b8", 8, 56, 64, 256, 1, 1, 0), ("stem b8", 8, 224, 4, 64, 7, 2, 3),
          ("l1.c2 b256", 256, 56, 64, 64, 3, 1, 1), ("l3.c2 b256", 256, 14, 256, 256, 3, 1, 1)]
for name, B, H, Cin, K, R, s, p in shapes:
    Ho = (H + 2 * p - R) // s + 1
    g = np.random.default_rng(0)
    x = g.standard_normal((B, H, H, Cin)).astype(np.float32)
    dy = g.standard_normal((B, Ho, Ho, K)).astype(np.float32)
    ref = None
    if B <= 8:
        ref = L.conv2d_wgrad(np.moveaxis(x, -1, 1).astype(np.float64), np.moveaxis(dy, -1, 1).astype(np.float64),
                             (K, Cin, R, R), s, p)          # [K, C, R, R]
        ref = np.moveaxis(ref, 1, -1)                        # KRSC
    xt, dyt = torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda()
    dw = torch.empty(K, R, R, Cin, device="cuda")
    for kmax in ("0", "256", "128", "64", "32"):
        os.environ["POOCH_WGRAD_KMAX"] = kmax
        d = _lib.ConvDesc(B, H, H, Cin, K, R, R, s, p, 1)
        wsb = _lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d))
        ws = torch.empty(max(wsb // 4, 1), device="cuda")
        f = lambda: _lib.lib.pooch_op_conv_wgrad(C.byref(d), P(xt), P(dyt), P(dw), P(ws), wsb, None)  # noqa: E731
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        err = None
        if ref is not None:
            got = dw.cpu().numpy().astype(np.float64)
            err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        print("%-12s kmax %-4s ws %8.1f MB  %.4f ms  rel-L2 %s" % (name, kmax, wsb / 1e6, ms,
                                                                     "%.2e" % err if err is not None else "-"), flush=True)
