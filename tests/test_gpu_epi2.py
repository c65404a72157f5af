"""Two epilogue warp groups (igemm.cuh E2, POOCH_EPI2) against the one-group epilogue: each group
drains half of the accumulator's columns through the same TMEM loads, staging, per-quadrant BN
partial sums (the same rows in the same order) and TMA stores, so y, the BN tile sums and dx
(plain and accumulating) must agree bit for bit -- 2D at tile widths 64 / 128, a strided
layer, a 3D conv. Subprocesses: the switch is read once per process."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [
    # N, H, W, C, K, R, stride, pad, D (0 = 2D)
    (2, 14, 14, 64, 64, 3, 1, 1, 0),
    (2, 14, 13, 64, 256, 1, 1, 0, 0),
    (2, 15, 13, 128, 128, 3, 2, 1, 0),
    (1, 8, 8, 32, 64, 3, 1, 1, 6),
]

SCRIPT = r"""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, %(root)r)
from paper_1907_05013_b200 import _lib as lib
N, H, W, Cc, K, R, s, p, D = %(case)r
d = lib.ConvDesc(N, H, W, Cc, K, R, R, s, p, 1, D, 0, 0, 0)
g = np.random.default_rng(sum(%(case)r))
Ho, Wo = (H + 2 * p - R) // s + 1, (W + 2 * p - R) // s + 1
Do = (D + 2 * p - R) // s + 1 if D else 1
T = R if D else 1
x = torch.from_numpy(g.standard_normal(N * max(D, 1) * H * W * Cc).astype(np.float32)).cuda()
w = torch.from_numpy((0.1 * g.standard_normal(K * T * R * R * Cc)).astype(np.float32)).cuda()
dy = torch.from_numpy(g.standard_normal(N * Do * Ho * Wo * K).astype(np.float32)).cuda()
wt = w.view(K, T * R * R, Cc).permute(2, 1, 0).contiguous().view(-1)
y = torch.full((N * Do * Ho * Wo * K,), float("nan"), device="cuda")
mt = lib.lib.pooch_op_conv_stat_tiles(C.byref(d))
s1 = torch.full((mt * K,), float("nan"), device="cuda")
s2 = torch.full((mt * K,), float("nan"), device="cuda")
dx = torch.full_like(x, float("nan"))
dxa = torch.from_numpy(g.standard_normal(x.numel()).astype(np.float32)).cuda()
P = lambda t: C.c_void_p(t.data_ptr())
lib.check(lib.lib.pooch_op_conv_fwd(C.byref(d), P(x), P(w), P(y), P(s1), P(s2), None))
lib.check(lib.lib.pooch_op_conv_dgrad(C.byref(d), P(dy), P(wt), P(dx), 0, None))
lib.check(lib.lib.pooch_op_conv_dgrad(C.byref(d), P(dy), P(wt), P(dxa), 1, None))
torch.cuda.synchronize()
np.savez(sys.argv[1], y=y.cpu().numpy(), s1=s1.cpu().numpy(), s2=s2.cpu().numpy(), dx=dx.cpu().numpy(),
         dxa=dxa.cpu().numpy())
"""


@pytest.mark.parametrize("case", CASES)
def test_two_epilogue_groups_equal_one(tmp_path, case):
    root = os.path.dirname(HERE)
    code = SCRIPT % {"root": root, "case": case}
    outs = []
    for e2 in ("2", "0"):
        f = str(tmp_path / ("o_%s.npz" % e2))
        env = dict(os.environ, POOCH_EPI2=e2, POOCH_W2="0")  # W2 (BN = 64) exists only with E2
        r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    for k in ("y", "s1", "s2", "dx", "dxa"):
        assert np.isfinite(outs[0][k]).all(), k
        assert np.array_equal(outs[0][k].view(np.uint32), outs[1][k].view(np.uint32)), k


STEM_SCRIPT = r"""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, %(root)r)
from paper_1907_05013_b200 import _lib as lib
N, H, W, K, R, s, p = %(case)r
d = lib.ConvDesc(N, H, W, 4, K, R, R, s, p, 1)
g = np.random.default_rng(sum(%(case)r))
Ho, Wo = (H + 2 * p - R) // s + 1, (W + 2 * p - R) // s + 1
x = torch.from_numpy(g.standard_normal(N * H * W * 4).astype(np.float32)).cuda()
w = torch.from_numpy((0.1 * g.standard_normal(K * R * R * 4)).astype(np.float32)).cuda()
y = torch.full((N * Ho * Wo * K,), float("nan"), device="cuda")
mt = lib.lib.pooch_op_conv_stat_tiles(C.byref(d))
s1 = torch.full((mt * K,), float("nan"), device="cuda")
s2 = torch.full((mt * K,), float("nan"), device="cuda")
P = lambda t: C.c_void_p(t.data_ptr())
lib.check(lib.lib.pooch_op_conv_fwd(C.byref(d), P(x), P(w), P(y), P(s1), P(s2), None))
torch.cuda.synchronize()
np.savez(sys.argv[1], y=y.cpu().numpy(), s1=s1.cpu().numpy().reshape(mt, K).astype(np.float64).sum(0))
"""


@pytest.mark.parametrize("case", [(3, 224, 224, 64, 7, 2, 3), (2, 50, 46, 64, 7, 2, 3), (4, 32, 32, 32, 3, 1, 1)])
def test_patch_stem_equals_gather_stem(tmp_path, case):
    """The patch-gather stem (igemm.cuh SP, with three N = 64 MMAs per k-step) sums the same TF32
    products in the same K order per output element as the cp.async gather kernel, so y must be
    bit-identical (the BN tile partition differs, so only the tile sums' totals are compared)."""
    root = os.path.dirname(HERE)
    code = STEM_SCRIPT % {"root": root, "case": case}
    outs = []
    for on in ("1", "0"):
        f = str(tmp_path / ("o_%s.npz" % on))
        env = dict(os.environ, POOCH_STEM_PATCH=on, POOCH_W2="0")  # W2 sums the products differently
        r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    assert np.isfinite(outs[0]["y"]).all()
    assert np.array_equal(outs[0]["y"].view(np.uint32), outs[1]["y"].view(np.uint32))
    a, b = outs[0]["s1"], outs[1]["s1"]
    assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max() + 1e-6
