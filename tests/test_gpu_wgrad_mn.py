"""The transpose-free wgrad (MN-major tf32 operands, igemm.cuh MNW)
against the transposing kernels it replaced (POOCH_WGRAD_MN=0, run in a subprocess since the
switch is read once per process): the same TF32 operand values reach the same MMAs in the same
K order, so dW must agree bit for bit -- 2D layers at BN = 64 (the swapped orientation) and
BN = 128, a strided layer, and a 3D conv, in 3xTF32 and TF32."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [
    # N, H, W, C, K, R, stride, pad, D (0 = 2D), precision
    (2, 14, 14, 64, 64, 3, 1, 1, 0, 1),
    (2, 14, 14, 128, 256, 1, 1, 0, 0, 1),
    (2, 15, 13, 64, 128, 3, 2, 1, 0, 1),
    (1, 8, 8, 32, 64, 3, 1, 1, 6, 1),
    (2, 14, 14, 64, 64, 3, 1, 1, 0, 0),
]

SCRIPT = r"""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, %(root)r)
from paper_1907_05013_b200 import _lib as lib
N, H, W, Cc, K, R, s, p, D, prec = %(case)r
d = lib.ConvDesc(N, H, W, Cc, K, R, R, s, p, prec, D, 0, 0, 0)
g = np.random.default_rng(sum(%(case)r))
Ho, Wo = (H + 2 * p - R) // s + 1, (W + 2 * p - R) // s + 1
Do = (D + 2 * p - R) // s + 1 if D else 1
x = torch.from_numpy(g.standard_normal(N * max(D, 1) * H * W * Cc).astype(np.float32)).cuda()
dy = torch.from_numpy(g.standard_normal(N * Do * Ho * Wo * K).astype(np.float32)).cuda()
dw = torch.full((K * R * R * (R if D else 1) * Cc,), float("nan"), device="cuda")
wsb = lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d))
ws = torch.empty(max(wsb // 4, 1), device="cuda")
P = lambda t: C.c_void_p(t.data_ptr())
lib.check(lib.lib.pooch_op_conv_wgrad(C.byref(d), P(x), P(dy), P(dw), P(ws), wsb, None))
torch.cuda.synchronize()
np.save(sys.argv[1], dw.cpu().numpy())
"""


@pytest.mark.parametrize("case", CASES)
def test_mn_major_wgrad_equals_transposing_wgrad(tmp_path, case):
    root = os.path.dirname(HERE)
    code = SCRIPT % {"root": root, "case": case}
    outs = []
    for mn in ("1", "0"):
        f = str(tmp_path / ("dw_%s.npy" % mn))
        # W2 (two N = 128 MMAs over [B; Bs] at BN = 64) sums A*B and A*Bs separately: off here, so the
        # comparison isolates the operand layout (W2 itself: oracle parity in test_gpu_ops)
        env = dict(os.environ, POOCH_WGRAD_MN=mn, POOCH_WGRAD_W2="0")
        r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    assert np.isfinite(outs[0]).all()
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
