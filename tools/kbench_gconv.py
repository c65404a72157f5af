"""Time the grouped conv3d passes (gconv.cu) at ResNeXt-101 (3D)'s shapes for a 64 x 512 x 512
input, against the FP32 ALU roof (148 SMs x 128 FMA/clk x 2 flop x the SM clock).

Run on the GPU box: python tools/kbench_gconv.py [out.json]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch  # noqa: E402

from paper_1907_05013_b200 import _lib  # noqa: E402

SHAPES = [  # name, D, H, W (input), C, stride
    ("layer1.x.conv2", 32, 128, 128, 128, 1),
    ("layer2.0.conv2", 32, 128, 128, 256, 2),
    ("layer2.x.conv2", 16, 64, 64, 256, 1),
    ("layer3.0.conv2", 16, 64, 64, 512, 2),
    ("layer3.x.conv2", 8, 32, 32, 512, 1),
    ("layer4.0.conv2", 8, 32, 32, 1024, 2),
    ("layer4.x.conv2", 4, 16, 16, 1024, 1),
]


def clock_mhz():
    try:
        import subprocess
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.max.sm", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.split()
        return float(out[0])
    except Exception:
        return 1965.0


REPS = int(os.environ.get("POOCH_KB_REPS", "10"))
PICK = [int(v) for v in os.environ.get("POOCH_KB_SHAPES", "").split(",") if v]


def timeit(fn, reps=REPS):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    lib = _lib
    peak = 148 * 128 * 2 * clock_mhz() * 1e6 / 1e12
    rows = []
    for si, (name, D, H, W, Cc, s) in enumerate(SHAPES):
        if PICK and si not in PICK:
            continue
        d = lib.ConvDesc(1, H, W, Cc, Cc, 3, 3, s, 1, 1, D, 0, 32, 0)
        Do, Ho, Wo = (D - 1) // s + 1, (H - 1) // s + 1, (W - 1) // s + 1
        x = torch.randn(D * H * W * Cc, device="cuda")
        w = torch.randn(Cc * 27 * (Cc // 32), device="cuda")
        y = torch.empty(Do * Ho * Wo * Cc, device="cuda")
        mt = lib.lib.pooch_op_conv_stat_tiles(C.byref(d))
        s1, s2 = torch.empty(mt * Cc, device="cuda"), torch.empty(mt * Cc, device="cuda")
        wsb = lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d))
        ws = torch.empty(max(wsb // 4, 1), device="cuda")
        gw = torch.empty_like(w)
        gx = torch.empty_like(x)
        P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        flops = 2.0 * Do * Ho * Wo * Cc * 27 * (Cc // 32)
        t_f = timeit(lambda: lib.lib.pooch_op_conv_fwd(C.byref(d), P(x), P(w), P(y), P(s1), P(s2), None))
        t_d = timeit(lambda: lib.lib.pooch_op_conv_dgrad(C.byref(d), P(y), P(w), P(gx), 0, None))
        t_w = timeit(lambda: lib.lib.pooch_op_conv_wgrad(C.byref(d), P(x), P(y), P(gw), P(ws), wsb, None))
        r = {"layer": name, "C": Cc, "per_group": Cc // 32, "stride": s, "gflop": flops / 1e9,
             "fwd_ms": t_f, "dgrad_ms": t_d, "wgrad_ms": t_w,
             "fwd_frac": flops / (t_f * 1e-3) / 1e12 / peak, "dgrad_frac": flops / (t_d * 1e-3) / 1e12 / peak,
             "wgrad_frac": flops / (t_w * 1e-3) / 1e12 / peak}
        rows.append(r)
        print("%-16s C %4d  %.1f GFLOP  fwd %.3f ms (%.2f)  dgrad %.3f ms (%.2f)  wgrad %.3f ms (%.2f)" % (
            name, Cc, r["gflop"], t_f, r["fwd_frac"], t_d, r["dgrad_frac"], t_w, r["wgrad_frac"]), flush=True)
    out = {"peak_fp32_tflops": peak, "rows": rows}
    if len(sys.argv) > 1:
        json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
