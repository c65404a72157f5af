"""Accuracy of long wgrad splits (tensor-core accumulation bias, DESIGN.md Reading 43) at the lengths
the benchmark batches would produce without the split cap: dW rel-L2 against fp64 for a forced split
count (POOCH_WGRAD_SPLITS, cap off) and for the default cap (2048 k-blocks) and 1024.
Each case runs in its own process (the switches are read by the library). GPU box:
    python tools/acc_split_probe.py > gpurun_out/acc_split_probe.log
"""
import os
import subprocess
import sys

CASES = [  # name, B, H, Cin, K, R, stride, pad
    ("stem b32", 32, 224, 4, 64, 7, 2, 3),
    ("l1.c2 b32", 32, 56, 64, 64, 3, 1, 1),
]
SETTINGS = [("default cap (2048)", {}), ("cap 1024", {"POOCH_WGRAD_KMAX": "1024"}), ("no cap, 8 splits", {"POOCH_WGRAD_KMAX": "0", "POOCH_WGRAD_SPLITS": "8"}),
            ("no cap, 2 splits", {"POOCH_WGRAD_KMAX": "0", "POOCH_WGRAD_SPLITS": "2"}),
            ("no cap, 1 split", {"POOCH_WGRAD_KMAX": "0", "POOCH_WGRAD_SPLITS": "1"})]

CHILD = r"""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1907_05013_b200 import _lib
name, B, H, Cin, K, R, s, p = %(case)r
Ho = (H + 2 * p - R) // s + 1
g = np.random.default_rng(0)
x = g.standard_normal((B, H, H, Cin)).astype(np.float32)
dy = g.standard_normal((B, Ho, Ho, K)).astype(np.float32)
d = _lib.ConvDesc(B, H, H, Cin, K, R, R, s, p, 1)
wsb = _lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d))
ws = torch.empty(max(wsb // 4, 1), device="cuda")
xt, dyt = torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda()
dw = torch.empty(K, R, R, Cin, device="cuda")
P = lambda t: C.c_void_p(t.data_ptr())
_lib.check(_lib.lib.pooch_op_conv_wgrad(C.byref(d), P(xt), P(dyt), P(dw), P(ws), wsb, None))
torch.cuda.synchronize()
got = dw.cpu().numpy().astype(np.float64)
# fp64 reference: dW[k, r, s, c] = sum over pixels of dy[n, i, j, k] * xpad[n, s*i + r, s*j + s', c]
xp = np.pad(x.astype(np.float64), ((0, 0), (p, p), (p, p), (0, 0)))
dy64 = dy.reshape(-1, K).astype(np.float64)
ref = np.empty((K, R, R, Cin))
for r in range(R):
    for q in range(R):
        patch = xp[:, r:r + s * (Ho - 1) + 1:s, q:q + s * (Ho - 1) + 1:s, :].reshape(-1, Cin)
        ref[:, r, q, :] = dy64.T @ patch
err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
print("%%.3e %%d" %% (err, wsb))
"""

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for case in CASES:
    npx = case[1] * ((case[2] + 2 * case[7] - case[5]) // case[6] + 1) ** 2
    for label, env in SETTINGS:
        r = subprocess.run([sys.executable, "-c", CHILD % {"case": case}], env=dict(os.environ, **env), cwd=root,
                           capture_output=True, text=True, timeout=900)
        out = r.stdout.strip() or r.stderr.strip()[-300:]
        print("%-10s %7d pixels  %-20s rel-L2 / ws bytes: %s" % (case[0], npx, label, out), flush=True)
