"""Measure the divided layer (divide.cu) at a size whose maps exceed its device
workspace: conv3d 3^3 (C -> K) + BN + ReLU over an E^3 volume, forward (conv + statistics, BN-ReLU
apply) and backward (BN-ReLU two-pass, dgrad, wgrad), host-resident tensors, against the same
kernels run undivided on device-resident tensors, and against the host link (the layer is bound
by it: every byte of every map crosses PCIe once per pass).

Run on the GPU box: python tools/bench_divide.py [E] [C] [K] [ws_MiB] [out.json]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1907_05013_b200 import _lib  # noqa: E402


def main():
    E = int(sys.argv[1]) if len(sys.argv) > 1 else 192
    Cc = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    ws_mib = int(sys.argv[4]) if len(sys.argv) > 4 else 512
    out = sys.argv[5] if len(sys.argv) > 5 else None
    lib = _lib
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    d = lib.ConvDesc(1, E, E, Cc, K, 3, 3, 1, 1, 1, E, 0, 0, 0)
    nx, ny = E ** 3 * Cc, E ** 3 * K
    g = torch.Generator().manual_seed(0)
    xh = torch.randn(nx, generator=g).pin_memory()
    yh = torch.empty(ny).pin_memory()
    rh = torch.empty(ny).pin_memory()
    gyh = torch.randn(ny, generator=g).pin_memory()
    gch = torch.empty(ny).pin_memory()
    gxh = torch.empty(nx).pin_memory()
    w = (torch.randn(K * 27 * Cc, generator=g) / np.sqrt(27 * Cc)).cuda()
    wt = w.view(K, 27, Cc).permute(2, 1, 0).contiguous()
    gam, bet = torch.ones(K, device="cuda"), torch.zeros(K, device="cuda")
    stats = torch.empty(4 * K, device="cuda")
    dg, db = torch.empty(K, device="cuda"), torch.empty(K, device="cuda")
    dw = torch.empty_like(w)
    wsb = ws_mib << 20
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    ss = [torch.cuda.Stream() for _ in range(3)]
    sarr = (C.c_void_p * 3)(*[C.c_void_p(s.cuda_stream) for s in ss])
    res = {"volume": E, "C": Cc, "K": K, "workspace_bytes": wsb, "map_bytes_in": 4 * nx, "map_bytes_out": 4 * ny}

    def run(name, fn):
        info = lib.DivInfo()
        lib.check(fn(C.byref(info)))        # warm-up
        info = lib.DivInfo()
        lib.check(fn(C.byref(info)))
        gbs = (info.h2d_bytes + info.d2h_bytes) / (info.ms * 1e6)
        res[name] = {"ms": info.ms, "chunks": info.chunks, "rows_per_chunk": info.rows_per_chunk,
                     "h2d_bytes": info.h2d_bytes, "d2h_bytes": info.d2h_bytes, "h2d_gbs": info.h2d_bytes / (info.ms * 1e6),
                     "d2h_gbs": info.d2h_bytes / (info.ms * 1e6), "link_gbs": gbs}
        print(name, json.dumps(res[name]), flush=True)

    run("conv_fwd", lambda i: lib.lib.pooch_div_conv3d_fwd(C.byref(d), P(xh), P(w), P(yh), P(gam), P(bet), P(stats),
                                                            P(ws), wsb, sarr, i))
    run("bn_relu_fwd", lambda i: lib.lib.pooch_div_bn_relu_fwd(P(yh), P(stats), P(rh), E, E * E * K, K, P(ws), wsb,
                                                                sarr, i))
    run("bn_relu_bwd", lambda i: lib.lib.pooch_div_bn_relu_bwd(P(yh), P(gyh), P(stats), P(gam), P(dg), P(db), P(gch),
                                                                E, E * E * K, K, P(ws), wsb, sarr, i))
    run("conv_dgrad", lambda i: lib.lib.pooch_div_conv3d_dgrad(C.byref(d), P(gch), P(wt), P(gxh), P(ws), wsb, sarr,
                                                                i))
    run("conv_wgrad", lambda i: lib.lib.pooch_div_conv3d_wgrad(C.byref(d), P(xh), P(gch), P(dw), P(ws), wsb, sarr,
                                                                i))
    # the same kernels undivided, device-resident (the layer's compute alone)
    del ws
    torch.cuda.empty_cache()
    xd, yd, gd = xh.cuda(), torch.empty(ny, device="cuda"), gch.cuda()
    gx = torch.empty(nx, device="cuda")
    mt = lib.lib.pooch_op_conv_stat_tiles(C.byref(d))
    s1, s2 = torch.empty(mt * K, device="cuda"), torch.empty(mt * K, device="cuda")
    wsw = lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d))
    wws = torch.empty(max(wsw // 4, 1), device="cuda")

    def t(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    res["incore_kernels_ms"] = {
        "conv_fwd": t(lambda: lib.lib.pooch_op_conv_fwd(C.byref(d), P(xd), P(w), P(yd), P(s1), P(s2), None)),
        "conv_dgrad": t(lambda: lib.lib.pooch_op_conv_dgrad(C.byref(d), P(gd), P(wt), P(gx), 0, None)),
        "conv_wgrad": t(lambda: lib.lib.pooch_op_conv_wgrad(C.byref(d), P(xd), P(gd), P(dw), P(wws), wsw, None)),
    }
    torch.cuda.synchronize()
    res["fwd_bitexact_vs_undivided"] = bool(torch.equal(yd.cpu(), yh))
    print(json.dumps(res["incore_kernels_ms"]), "fwd bit-exact", res["fwd_bitexact_vs_undivided"], flush=True)
    if out:
        json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
