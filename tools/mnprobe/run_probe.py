"""Run the MN-major tf32 probe (tools/mnprobe/mnprobe.cu) for a few descriptor variants and
report which reproduces A^T B (fp64 reference of TF32-truncated operands). GPU box only."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "mnprobe.so")
if not os.path.exists(so):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
                           "-shared", "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "mnprobe.cu"), "-lcuda"])
lib = C.CDLL(so)
lib.mnprobe_run.argtypes = [C.c_void_p] * 3 + [C.c_uint32] * 4 + [C.c_int] * 2
lib.mnprobe_halo.argtypes = [C.c_void_p] * 3 + [C.c_uint32] * 2

K, M, N = 32, 128, 128
g = np.random.default_rng(0)
a = g.standard_normal((K, M)).astype(np.float32)
b = g.standard_normal((K, N)).astype(np.float32)


def tf32_trunc(x):
    return (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


ref = tf32_trunc(a).astype(np.float64).T @ tf32_trunc(b).astype(np.float64)   # [M][N]
da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
dd = torch.zeros((M, N), device="cuda")
# swz: 4 = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 3 = SWIZZLE_128B; layout: 1 = SW128_BASE32B, 2 = SW128
for name, lbo, sbo, layout, swz in [
        ("SW128_32B lbo=4096 sbo=512", 4096, 512, 1, 4),
        ("SW128_32B lbo=512 sbo=4096", 512, 4096, 1, 4),
        ("SW128 lbo=4096 sbo=1024", 4096, 1024, 2, 3),
        ("SW128 lbo=1024 sbo=4096", 1024, 4096, 2, 3)]:
    dd.zero_()
    rc = lib.mnprobe_run(C.c_void_p(da.data_ptr()), C.c_void_p(db.data_ptr()), C.c_void_p(dd.data_ptr()),
                         lbo, sbo, lbo, sbo, layout, swz)
    out = dd.cpu().numpy().astype(np.float64)
    err = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    print("%-30s rc %d  rel err %.3e  |D| %.3e" % (name, rc, err, np.linalg.norm(out)), flush=True)

# probe 2: A chunk q = the 40-row halo shifted by q (+ start) rows (LBO = 128 B)
halo = g.standard_normal((40, 32)).astype(np.float32)
dh = torch.from_numpy(halo).cuda()
for start in (0, 1, 2, 3, 5):
    A = np.zeros((M, K))
    for q in range(4):
        A[q * 32:(q + 1) * 32, :] = tf32_trunc(halo[start + q:start + q + K, :]).T.astype(np.float64)
    ref2 = A @ tf32_trunc(b).astype(np.float64)
    dd.zero_()
    rc = lib.mnprobe_halo(C.c_void_p(dh.data_ptr()), C.c_void_p(db.data_ptr()), C.c_void_p(dd.data_ptr()), 128, start)
    out = dd.cpu().numpy().astype(np.float64)
    print("halo start %d LBO 128: rc %d  rel err %.3e" % (start, rc, np.linalg.norm(out - ref2) / np.linalg.norm(ref2)),
          flush=True)
