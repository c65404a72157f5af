"""tcgen05.mma kind::tf32 throughput by tile width and A source (tools/mmaprobe/mmaprobe.cu)."""
import ctypes as C
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "mmaprobe.so")
if not os.path.exists(so):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
                           "-shared", "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "mmaprobe.cu")])
lib = C.CDLL(so)
lib.mmaprobe_run.restype = C.c_float
lib.mmaprobe_run.argtypes = [C.c_int, C.c_int, C.c_void_p]
cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
iters = 20000
for which, (n, src) in enumerate([(64, "smem"), (128, "smem"), (256, "smem"), (64, "tmem"), (128, "tmem"), (256, "tmem")]):
    ms = lib.mmaprobe_run(which, iters, C.c_void_p(cyc.data_ptr()))
    flops = 148 * iters * 2 * 128 * n * 8
    c = cyc.float().mean().item()
    print("N=%3d A in %s: %.3f ms  %.1f TFLOP/s (tf32)  %.1f cycles per MMA" % (n, src, ms, flops / ms / 1e9, c / iters),
          flush=True)
for which, n in [(6, 64), (7, 128)]:
    ms = lib.mmaprobe_run(which, iters, C.c_void_p(cyc.data_ptr()))
    flops = 148 * (iters // 12) * 12 * 2 * 128 * n * 8
    c = cyc.float().mean().item()
    print("k-block pattern N=%3d (lo*B, hi*Bs, hi*B, A in TMEM, commit per 12): %.3f ms  %.1f TFLOP/s  %.1f cycles per MMA"
          % (n, ms, flops / ms / 1e9, c / ((iters // 12) * 12)), flush=True)
for which, n, desc in [(8, 64, "6 stages, 128 arrivals"), (9, 64, "6 stages, 1 arrival"), (10, 64, "3 stages"),
                       (11, 128, "3 stages"), (12, 64, "2 stages"), (13, 64, "6 st, no fence"),
                       (14, 64, "6 st, lane-0 wait"), (15, 64, "6 st, both"), (16, 64, "6 st, no real wait"),
                       (17, 64, "6 st, suspend hint 32"), (18, 128, "3 st, no real wait"),
                       (19, 64, "no wait, idle consumers"), (20, 64, "+ no fence"), (21, 64, "+ no syncwarp"),
                       (22, 64, "no wait, no syncwarp")]:
    ms = lib.mmaprobe_run(which, iters, C.c_void_p(cyc.data_ptr()))
    flops = 148 * (iters // 12) * 12 * 2 * 128 * n * 8
    c = cyc.float().mean().item()
    print("ring N=%3d %-24s: %.3f ms  %.1f TFLOP/s  %.1f cycles per MMA" % (n, desc, ms, flops / ms / 1e9,
                                                                           c / ((iters // 12) * 12)), flush=True)
for which, desc in [(23, "try_wait per k-block"), (24, "commit to 6 rotating barriers"), (25, "fence per k-block"),
                    (26, "all three"), (27, "test_wait per k-block"), (28, "ld.shared of the barrier"),
                    (29, "try_wait after 6 of 12 MMAs")]:
    ms = lib.mmaprobe_run(which, iters, C.c_void_p(cyc.data_ptr()))
    c = cyc.float().mean().item()
    print("k-block pattern N= 64 %-30s: %.3f ms  %.1f cycles per MMA" % (desc, ms, c / ((iters // 12) * 12)), flush=True)
for which, desc in [(30, "try_wait per k-block"), (31, "no wait")]:
    ms = lib.mmaprobe_run(which, iters, C.c_void_p(cyc.data_ptr()))
    c = cyc.float().mean().item()
    print("k-block pattern N=128 %-30s: %.3f ms  %.1f cycles per MMA" % (desc, ms, c / ((iters // 12) * 12)), flush=True)
for which, desc in [(32, "merged hi*[B;Bs] N=128 + lo*B"), (33, "merged + try_wait per k-block"),
                    (34, "hi*[B;Bs] + lo*[B;Bs], both N=128"), (35, "both N=128 + try_wait")]:
    ms = lib.mmaprobe_run(which, iters, C.c_void_p(cyc.data_ptr()))
    c = cyc.float().mean().item()
    nk = iters // 12
    print("k-block N=64 %-36s: %.3f ms  %.1f cycles per k-block (12 N=64 MMAs' work)" % (desc, ms, c / nk), flush=True)
