"""GPU parity of the tensor-core implicit-GEMM passes against the fp64 oracle.

Each case runs one kernel through the C ABI (pooch_op_*) on cuda:0 and
compares every output element with oracle/layers.py (relative L2 error; TF32
inputs with fp32 accumulation, tolerance derived in DESIGN.md "Tolerances")."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import synthdata  # noqa: E402
from oracle import layers as L  # noqa: E402

TOL_OP = 3e-3
TOL_X3 = 2e-5     # 3xTF32 split: ~fp32 accumulation error at K <~ 2000 ...


def tol_x3(K):
    """... growing ~linearly with the reduction length: the tensor core's accumulation bias
    (Reading 43; test_3xtf32_error_against_fp32 measures 3.3e-5 at K = 4608)."""
    return max(TOL_X3, 1e-8 * K)


def _lib():
    from paper_1907_05013_b200 import _lib
    return _lib


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def ptr(t):
    return C.c_void_p(t.data_ptr())


@pytest.mark.parametrize("M,N,K,amn,bmn,bn,splits", [
    (128, 64, 32, 0, 0, 64, 1), (256, 128, 96, 0, 0, 128, 1), (300, 200, 100, 0, 0, 256, 1),
    (260, 136, 72, 0, 0, 128, 1), (384, 256, 520, 0, 0, 256, 3), (132, 1000, 2048, 0, 0, 256, 1),
    (256, 64, 64, 0, 0, 64, 2), (4096, 512, 1024, 0, 0, 256, 1),
    (300, 200, 100, 2, 0, 128, 1), (4096, 512, 1024, 2, 0, 128, 1)])
def test_gemm_core(M, N, K, amn, bmn, bn, splits):
    lib = _lib()
    g = synthdata.rng(M * 7 + N + K)
    A = g.standard_normal((M, K)).astype(np.float32)
    B = g.standard_normal((N, K)).astype(np.float32)
    dA = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    dB = torch.from_numpy(np.ascontiguousarray(B)).cuda()
    dD = torch.zeros((splits, M, N), dtype=torch.float32, device="cuda")
    lib.check(lib.lib.pooch_op_gemm_test(ptr(dA), ptr(dB), ptr(dD), M, N, K, amn, bmn, bn, splits, None))
    torch.cuda.synchronize()
    D = dD.cpu().numpy().astype(np.float64).sum(0)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    assert rel(D, ref) < (TOL_X3 if amn == 2 else TOL_OP)


CONV_CASES = [
    # N, H, W, C, K, R, stride, pad   (ResNet-50 / tiny-CNN shapes, shrunk spatially)
    (2, 16, 16, 4, 64, 7, 2, 3),      # stem (Cin padded 3->4)
    (2, 50, 46, 4, 64, 7, 2, 3),      # stem, several ragged 16 x 8 output boxes (patch-gather kernel)
    (2, 224, 224, 4, 64, 7, 2, 3),    # stem at full resolution (patch wgrad: 16 x 2 pixel boxes, split-K)
    (2, 8, 8, 64, 64, 1, 1, 0),       # 1x1
    (2, 8, 8, 64, 64, 3, 1, 1),       # 3x3
    (2, 9, 9, 128, 128, 3, 2, 1),     # strided 3x3, ragged
    (3, 7, 7, 256, 512, 1, 2, 0),     # projection 1x1 stride 2
    (8, 32, 32, 4, 32, 3, 1, 1),      # tiny CNN first conv
    (8, 32, 32, 32, 32, 3, 1, 1),     # tiny CNN conv
    (1, 5, 5, 512, 2048, 1, 1, 0),    # wide 1x1, M < 128
    (3, 6, 6, 256, 64, 1, 1, 0),      # 1x1 reduce to 64 (wgrad: transposed orientation)
    (2, 6, 6, 64, 256, 1, 1, 0),      # 1x1 expand from 64 (wgrad: 64-wide B tile)
    (5, 7, 7, 64, 96, 3, 1, 1),       # odd batch, ragged pixel boxes
    (2, 67, 67, 4, 96, 11, 4, 0),     # AlexNet conv1 (11x11 stride 4, Cin padded 3->4)
    (2, 13, 13, 96, 256, 5, 1, 2),    # AlexNet conv2 shape (5x5 pad 2), 96 channels
]


def _conv_inputs(N, H, W, Cin, K, R, seed):
    g = synthdata.rng(seed)
    x = g.standard_normal((N, H, W, Cin)).astype(np.float32)
    w = (g.standard_normal((K, R, R, Cin)) / np.sqrt(R * R * Cin)).astype(np.float32)
    return x, w


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_fwd_and_stats(case, prec):
    lib = _lib()
    N, H, W, Cin, K, R, s, p = case
    x, w = _conv_inputs(N, H, W, Cin, K, R, sum(case))
    d = lib.ConvDesc(N, H, W, Cin, K, R, R, s, p, prec)
    ho, wo = L.conv_out_hw(H, W, R, R, s, p)
    M = N * ho * wo
    mt = lib.lib.pooch_op_conv_stat_tiles(C.byref(d))
    dx, dw = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    dy = torch.full((N, ho, wo, K), float("nan"), device="cuda")
    s1 = torch.zeros((mt, K), device="cuda")
    s2 = torch.zeros((mt, K), device="cuda")
    lib.check(lib.lib.pooch_op_conv_fwd(C.byref(d), ptr(dx), ptr(dw), ptr(dy), ptr(s1), ptr(s2), None))
    torch.cuda.synchronize()
    ref = L.conv2d_fwd(x.transpose(0, 3, 1, 2).astype(np.float64), w.transpose(0, 3, 1, 2).astype(np.float64), s, p)
    ref = ref.transpose(0, 2, 3, 1)
    y = dy.cpu().numpy()
    assert rel(y, ref) < (tol_x3(R * R * Cin) if prec else TOL_OP)
    # per-tile partial sums add up to the column sums of y (checked against the oracle output)
    flat = ref.reshape(-1, K)
    assert rel(s1.cpu().numpy().astype(np.float64).sum(0), flat.sum(0)) < TOL_OP
    assert rel(s2.cpu().numpy().astype(np.float64).sum(0), (flat ** 2).sum(0)) < TOL_OP


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("accumulate", [0, 1])
def test_conv_dgrad(case, accumulate, prec):
    lib = _lib()
    N, H, W, Cin, K, R, s, p = case
    x, w = _conv_inputs(N, H, W, Cin, K, R, sum(case) + 1)
    ho, wo = L.conv_out_hw(H, W, R, R, s, p)
    gy = synthdata.rng(5).standard_normal((N, ho, wo, K)).astype(np.float32)
    prev = synthdata.rng(6).standard_normal((N, H, W, Cin)).astype(np.float32)
    wt = np.ascontiguousarray(w.transpose(3, 1, 2, 0))   # [C][R][S][K]
    d = lib.ConvDesc(N, H, W, Cin, K, R, R, s, p, prec)
    dgy, dwt = torch.from_numpy(gy).cuda(), torch.from_numpy(wt).cuda()
    ddx = torch.from_numpy(prev.copy()).cuda() if accumulate else torch.full((N, H, W, Cin), float("nan"), device="cuda")
    lib.check(lib.lib.pooch_op_conv_dgrad(C.byref(d), ptr(dgy), ptr(dwt), ptr(ddx), accumulate, None))
    torch.cuda.synchronize()
    ref = L.conv2d_dgrad(gy.transpose(0, 3, 1, 2).astype(np.float64), w.transpose(0, 3, 1, 2).astype(np.float64),
                         (N, Cin, H, W), s, p).transpose(0, 2, 3, 1)
    if accumulate:
        ref = ref + prev
    assert rel(ddx.cpu().numpy(), ref) < (tol_x3(R * R * K) if prec else TOL_OP)


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_wgrad(case, prec):
    lib = _lib()
    N, H, W, Cin, K, R, s, p = case
    x, w = _conv_inputs(N, H, W, Cin, K, R, sum(case) + 2)
    ho, wo = L.conv_out_hw(H, W, R, R, s, p)
    gy = synthdata.rng(7).standard_normal((N, ho, wo, K)).astype(np.float32)
    d = lib.ConvDesc(N, H, W, Cin, K, R, R, s, p, prec)
    wsb = lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d))
    ws = torch.empty(max(wsb // 4, 1), device="cuda")
    dx, dgy = torch.from_numpy(x).cuda(), torch.from_numpy(gy).cuda()
    ddw = torch.full((K, R, R, Cin), float("nan"), device="cuda")
    lib.check(lib.lib.pooch_op_conv_wgrad(C.byref(d), ptr(dx), ptr(dgy), ptr(ddw), ptr(ws), wsb, None))
    torch.cuda.synchronize()
    ref = L.conv2d_wgrad(x.transpose(0, 3, 1, 2).astype(np.float64), gy.transpose(0, 3, 1, 2).astype(np.float64),
                         (K, Cin, R, R), s, p).transpose(0, 2, 3, 1)
    assert rel(ddw.cpu().numpy(), ref) < (TOL_X3 if prec else TOL_OP)


def test_conv_large_wgrad_splitk():
    """A ResNet-50 stage-1 3x3 at batch 16 (M*K large enough to split K many ways)."""
    lib = _lib()
    N, H, W, Cin, K, R, s, p = 16, 56, 56, 64, 64, 3, 1, 1
    x, w = _conv_inputs(N, H, W, Cin, K, R, 11)
    gy = synthdata.rng(8).standard_normal((N, H, W, K)).astype(np.float32)
    d = lib.ConvDesc(N, H, W, Cin, K, R, R, s, p)
    wsb = lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d))
    assert wsb > 0
    ws = torch.empty(wsb // 4, device="cuda")
    ddw = torch.empty((K, R, R, Cin), device="cuda")
    dx, dgy = torch.from_numpy(x).cuda(), torch.from_numpy(gy).cuda()   # keep alive until synced
    lib.check(lib.lib.pooch_op_conv_wgrad(C.byref(d), ptr(dx), ptr(dgy), ptr(ddw), ptr(ws), wsb, None))
    torch.cuda.synchronize()
    ref = L.conv2d_wgrad(x.transpose(0, 3, 1, 2).astype(np.float64), gy.transpose(0, 3, 1, 2).astype(np.float64),
                         (K, Cin, R, R), s, p).transpose(0, 2, 3, 1)
    assert rel(ddw.cpu().numpy(), ref) < TOL_OP


@pytest.mark.parametrize("N,H,C,k,s,p", [
    (2, 9, 8, 3, 2, 1),      # ResNet stem pool shape class (k3 s2 p1), odd extent -> ragged windows
    (3, 16, 64, 3, 2, 1),
    (2, 12, 32, 2, 2, 0),    # tiny CNN (k2 s2)
    (1, 7, 4, 3, 1, 1)])     # overlapping stride-1 windows
def test_maxpool2d(N, H, C, k, s, p):
    """Max-pool fwd / bwd kernels vs the fp64 oracle (Sec. 2.1 layer math; Reading 25: gradient to
    the first maximum). Values are distinct per window except for the forced ties below, so the
    forward is exact and the backward routes every gradient to the same element as the oracle."""
    lib = _lib().lib
    g = synthdata.rng(11)
    x = g.standard_normal((N, C, H, H))
    x[:, :, 0, 0] = x[:, :, 0, 1]          # a tie: the first maximum must win on both sides
    y_ref = L.maxpool_fwd(x, k, s, p)
    gy = g.standard_normal(y_ref.shape)
    gx_ref = L.maxpool_bwd(gy, x, k, s, p)
    nhwc = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(0, 2, 3, 1), np.float32)).cuda()  # noqa: E731
    xd, gyd = nhwc(x), nhwc(gy)
    Ho = y_ref.shape[2]
    yd = torch.empty(N, Ho, Ho, C, device="cuda")
    gxd = torch.empty(N, H, H, C, device="cuda")
    ws = torch.empty(N * Ho * Ho * C, dtype=torch.uint8, device="cuda")
    assert lib.pooch_op_maxpool2d_fwd(ptr(xd), ptr(yd), N, H, H, C, k, s, p, None) == 0
    assert lib.pooch_op_maxpool2d_bwd(ptr(xd), ptr(gyd), ptr(gxd), ptr(ws), N, H, H, C, k, s, p, None) == 0
    torch.cuda.synchronize()
    y = yd.cpu().numpy().transpose(0, 3, 1, 2)
    gx = gxd.cpu().numpy().transpose(0, 3, 1, 2)
    np.testing.assert_array_equal(y, y_ref.astype(np.float32))
    assert rel(gx, gx_ref) < 1e-6
    # support of the routed gradient is identical (index work: exact)
    np.testing.assert_array_equal(gx != 0, gx_ref != 0)


BNRELU_CASES = [c for c in CONV_CASES if c[3] % 32 == 0 and c[6] <= 2] + [
    (4, 14, 14, 64, 64, 3, 1, 1),     # stage-1-like 3x3, several M tiles
    (3, 11, 11, 128, 64, 3, 2, 1),    # strided, ragged
]


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("case", BNRELU_CASES)
def test_conv_bnrelu_on_load(case, prec):
    """conv fwd and wgrad with the operand relu(scale * x + shift) rebuilt on load
    (pooch_op_conv_fwd_bnrelu / _wgrad_bnrelu) against the fp64 oracle conv of the stored
    relu(bn(.)) -- padding must stay zero (shift != 0 makes a wrong pad visible)."""
    lib = _lib()
    N, H, W, Cin, K, R, s, p = case
    x, w = _conv_inputs(N, H, W, Cin, K, R, sum(case) + 3)
    g = synthdata.rng(sum(case) + 4)
    scale = g.uniform(0.5, 1.5, Cin).astype(np.float32)
    shift = g.uniform(-0.5, 0.5, Cin).astype(np.float32)
    r = np.maximum(x.astype(np.float64) * scale + shift, 0.0)          # NHWC, fp64
    ho, wo = L.conv_out_hw(H, W, R, R, s, p)
    gy = g.standard_normal((N, ho, wo, K)).astype(np.float32)
    d = lib.ConvDesc(N, H, W, Cin, K, R, R, s, p, prec)
    mt = lib.lib.pooch_op_conv_stat_tiles(C.byref(d))
    dx, dw = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    dsc, dsh = torch.from_numpy(scale).cuda(), torch.from_numpy(shift).cuda()
    dy = torch.full((N, ho, wo, K), float("nan"), device="cuda")
    s1 = torch.zeros((mt, K), device="cuda")
    s2 = torch.zeros((mt, K), device="cuda")
    lib.check(lib.lib.pooch_op_conv_fwd_bnrelu(C.byref(d), ptr(dx), ptr(dsc), ptr(dsh), ptr(dw), ptr(dy), ptr(s1),
                                               ptr(s2), None))
    wsb = lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d))
    ws = torch.empty(max(wsb // 4, 1), device="cuda")
    dgy = torch.from_numpy(gy).cuda()
    ddw = torch.full((K, R, R, Cin), float("nan"), device="cuda")
    lib.check(lib.lib.pooch_op_conv_wgrad_bnrelu(C.byref(d), ptr(dx), ptr(dsc), ptr(dsh), ptr(dgy), ptr(ddw), ptr(ws),
                                                 wsb, None))
    torch.cuda.synchronize()
    rn = r.transpose(0, 3, 1, 2)
    ref = L.conv2d_fwd(rn, w.transpose(0, 3, 1, 2).astype(np.float64), s, p).transpose(0, 2, 3, 1)
    tol = TOL_X3 if prec else TOL_OP
    assert rel(dy.cpu().numpy(), ref) < tol
    flat = ref.reshape(-1, K)
    assert rel(s1.cpu().numpy().astype(np.float64).sum(0), flat.sum(0)) < TOL_OP
    refw = L.conv2d_wgrad(rn, gy.transpose(0, 3, 1, 2).astype(np.float64), (K, Cin, R, R), s, p).transpose(0, 2, 3, 1)
    assert rel(ddw.cpu().numpy(), refw) < tol


def _emulated_3xtf32(A, B):
    """The 3xTF32 products with EXACT (fp64) accumulation: hi = trunc_tf32(x), lo = trunc_tf32(x -
    hi) (the tensor core truncates both, DESIGN.md Reading 27), D = Ah Bh + Ah Bl + Al Bh."""
    t = lambda x: (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)
    ah, bh = t(A), t(B)
    al, bl = t(A - ah.astype(np.float32)), t(B - bh.astype(np.float32))
    return ah @ bh.T + ah @ bl.T + al @ bh.T


@pytest.mark.parametrize("K", [576, 4608, 32768])
def test_3xtf32_error_against_fp32(K):
    """How accurate the contraction kernels are next to plain fp32 (Reading 28 sets the gradient
    gate from this): rel-L2 vs fp64 of the GPU's 3xTF32 GEMM, of CPU fp32 BLAS on the same operands,
    and of the 3xTF32 products accumulated exactly (isolating the tensor core's accumulation)."""
    lib = _lib()
    g = synthdata.rng(K)
    M, N = 512, 256
    A = g.standard_normal((M, K)).astype(np.float32)
    B = g.standard_normal((N, K)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dD = torch.zeros((1, M, N), dtype=torch.float32, device="cuda")
    lib.check(lib.lib.pooch_op_gemm_test(ptr(dA), ptr(dB), ptr(dD), M, N, K, 2, 0, 128, 1, None))
    torch.cuda.synchronize()
    e_gpu = rel(dD.cpu().numpy()[0].astype(np.float64), ref)
    e_f32 = rel((A @ B.T).astype(np.float64), ref)
    e_emu = rel(_emulated_3xtf32(A, B), ref)
    print("\nK=%d: 3xTF32 GPU %.2e, fp32 BLAS %.2e, 3xTF32 products exactly accumulated %.2e (GPU / fp32 = %.1f)"
          % (K, e_gpu, e_f32, e_emu, e_gpu / e_f32))
    # the split itself is fp32-faithful (exact accumulation of the three TF32 products ~ fp32 BLAS);
    # the tensor core's accumulation adds an error ~linear in the number of accumulated MMAs
    # (measured 4.5e-6 / 3.3e-5 / 2.3e-4 at K = 576 / 4608 / 32768), bounded here at 1e-8 per k
    assert e_emu < 2 * e_f32
    assert e_gpu < max(TOL_X3, 1e-8 * K)
