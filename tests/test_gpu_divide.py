"""Intra-layer division (ooc_cuDNN style; Sec. 6) through the C ABI
(pooch_div_*): a conv3d -> BN -> ReLU layer run on host-resident tensors in chunks of depth rows
through a device workspace far smaller than its maps.

* conv3d forward and dgrad equal the undivided kernels (pooch_op_conv_*) bit for bit -- each
  output element is computed by the same kernel over the same taps (halo rows are real rows or
  the volume's zero faces); strides 1 and 2, ragged last chunks;
* the BN statistics, the BN-ReLU backward sums and wgrad regroup their sums over chunks: against
  the undivided launch within fp32 summation error and against the fp64 oracle within the
  3xTF32 / fp32 tolerances;
* the BN-ReLU apply equals the undivided kernel bit for bit;
* a workspace too small for one row is POOCH_EINFEASIBLE.
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthdata  # noqa: E402
from oracle import layers as L  # noqa: E402
from netutil import rel  # noqa: E402


def _lib():
    from paper_1907_05013_b200 import _lib
    return _lib


def ptr(t):
    return C.c_void_p(t.data_ptr())


def ndhwc(a):
    return np.ascontiguousarray(np.moveaxis(a, 1, -1))


def ncdhw(a):
    return np.moveaxis(a, -1, 1)


def pinned(a):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).pin_memory()
    return t


def host_empty(n):
    return torch.full((n,), float("nan"), dtype=torch.float32).pin_memory()


def _streams():
    ss = [torch.cuda.Stream() for _ in range(3)]
    arr = (C.c_void_p * 3)(*[C.c_void_p(s.cuda_stream) for s in ss])
    return ss, arr


def _chunked(lib, call, start_bytes, min_chunks=3):
    """Run call(ws_ptr, ws_bytes, info) with a workspace shrunk (x 0.7 per try) until the layer
    runs in >= min_chunks chunks; returns the info of that run (its outputs are the call's)."""
    nbytes = int(start_bytes)
    while nbytes > 4096:
        ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        info = lib.DivInfo()
        st = call(ptr(ws), nbytes, C.byref(info))
        if st == 2:
            break
        lib.check(st)
        if info.chunks >= min_chunks:
            return info
        nbytes = int(nbytes * 0.7)
    raise AssertionError("no workspace gives %d chunks" % min_chunks)


def _tol_x3(K):
    return max(2e-5, 1e-8 * K)


# D, H, W, C, K, k, stride; the workspace is half the layer's input + output bytes (+ the BN
# tile partials), so every pass runs in several chunks with a ragged last one
CASES = [
    (13, 10, 9, 32, 64, 3, 1),
    (14, 9, 11, 64, 32, 3, 2),
    (9, 8, 8, 32, 32, 1, 1),
]


@pytest.mark.parametrize("case", CASES)
def test_divided_conv_bn_relu_layer(case):
    lib = _lib()
    D, H, W, Cc, K, k, s = case
    p = k // 2
    g = synthdata.rng(sum(case) % 1000)
    x = g.standard_normal((1, Cc, D, H, W)).astype(np.float32).astype(np.float64)
    w = (g.standard_normal((K, Cc, k, k, k)) / np.sqrt(Cc * k ** 3)).astype(np.float32).astype(np.float64)
    gamma = g.uniform(0.5, 1.5, K).astype(np.float32)
    beta = g.uniform(-0.2, 0.2, K).astype(np.float32)
    d = lib.ConvDesc(1, H, W, Cc, K, k, k, s, p, 1, D, 0, 0, 0)
    y_ref = L.conv3d_fwd(x, w, s, p)
    Do, Ho, Wo = y_ref.shape[2:]
    wsb = (D * H * W * Cc + Do * Ho * Wo * K) * 4 // 2 + (64 << 10)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    ss, sarr = _streams()
    info = lib.DivInfo()
    dw_dev = torch.from_numpy(np.ascontiguousarray(np.moveaxis(w, 1, -1)).astype(np.float32)).cuda()
    gam, bet = torch.from_numpy(gamma).cuda(), torch.from_numpy(beta).cuda()
    stats = torch.full((4 * K,), float("nan"), device="cuda")
    xh = pinned(ndhwc(x))
    yh = host_empty(Do * Ho * Wo * K)
    # ---- conv fwd + BN statistics, divided
    lib.check(lib.lib.pooch_div_conv3d_fwd(C.byref(d), ptr(xh), ptr(dw_dev), ptr(yh), ptr(gam), ptr(bet), ptr(stats),
                                           ptr(ws), wsb, sarr, C.byref(info)))
    assert info.chunks >= 3, info.chunks
    # undivided launch of the same kernel: identical bits
    xd = xh.cuda()
    yd = torch.full((Do * Ho * Wo * K,), float("nan"), device="cuda")
    lib.check(lib.lib.pooch_op_conv_fwd(C.byref(d), ptr(xd), ptr(dw_dev), ptr(yd), None, None, None))
    torch.cuda.synchronize()
    assert torch.equal(yh, yd.cpu()), "divided conv fwd differs from the undivided kernel"
    assert rel(ncdhw(yh.numpy().reshape(1, Do, Ho, Wo, K)), y_ref) < _tol_x3(Cc * k ** 3)
    # statistics against fp64 of the same y
    yv = yh.numpy().reshape(-1, K).astype(np.float64)
    mu, var = yv.mean(0), yv.var(0)
    st = stats.cpu().numpy()
    assert np.max(np.abs(st[:K] - mu)) < 1e-5 * max(1.0, np.abs(mu).max())
    assert rel(st[K:2 * K], 1.0 / np.sqrt(var + 1e-5)) < 1e-5
    # ---- BN-ReLU apply: equal to the undivided kernel
    rh = host_empty(yh.numel())
    lib.check(lib.lib.pooch_div_bn_relu_fwd(ptr(yh), ptr(stats), ptr(rh), Do, Ho * Wo * K, K, ptr(ws), wsb, sarr,
                                            C.byref(info)))
    rd = torch.empty_like(yd)
    lib.check(lib.lib.pooch_op_bn_relu_fwd(ptr(yd), ptr(stats[2 * K:]), ptr(stats[3 * K:]), ptr(rd), yd.numel() // K,
                                           K, None))
    torch.cuda.synchronize()
    assert torch.equal(rh, rd.cpu())
    # ---- BN-ReLU backward (two passes over the chunks) against the undivided kernel and the oracle
    gy = synthdata.rng(7).standard_normal(yh.numel()).astype(np.float32)
    gyh = pinned(gy)
    dg, db = torch.zeros(K, device="cuda"), torch.zeros(K, device="cuda")
    gch = host_empty(yh.numel())
    lib.check(lib.lib.pooch_div_bn_relu_bwd(ptr(yh), ptr(gyh), ptr(stats), ptr(gam), ptr(dg), ptr(db), ptr(gch), Do,
                                            Ho * Wo * K, K, ptr(ws), wsb, sarr, C.byref(info)))
    bws = torch.empty(lib.lib.pooch_op_bn_ws_bytes(K), dtype=torch.uint8, device="cuda")
    dg2, db2 = torch.zeros(K, device="cuda"), torch.zeros(K, device="cuda")
    gcd = torch.empty_like(yd)
    gyd = gyh.cuda()
    lib.check(lib.lib.pooch_op_bn_relu_bwd(ptr(yd), ptr(gyd), ptr(stats[2 * K:]), ptr(stats[3 * K:]), ptr(stats),
                                           ptr(stats[K:]), ptr(gam), ptr(dg2), ptr(db2), ptr(gcd), yd.numel() // K, K,
                                           ptr(bws), None))
    torch.cuda.synchronize()
    assert rel(gch.numpy(), gcd.cpu().numpy()) < 1e-5
    assert rel(dg.cpu().numpy(), dg2.cpu().numpy()) < 1e-5 and rel(db.cpu().numpy(), db2.cpu().numpy()) < 1e-5
    c64 = ncdhw(yv.reshape(1, Do, Ho, Wo, K))
    z, cache = L.bn_fwd(c64, gamma.astype(np.float64), beta.astype(np.float64))
    dz = L.relu_bwd(ncdhw(gy.astype(np.float64).reshape(1, Do, Ho, Wo, K)), L.relu_fwd(z))
    dx_ref, dg_ref, db_ref = L.bn_bwd(dz, cache, gamma.astype(np.float64))
    assert rel(ncdhw(gch.numpy().reshape(1, Do, Ho, Wo, K)), dx_ref) < 1e-4
    assert rel(dg.cpu().numpy(), dg_ref) < 1e-4 and rel(db.cpu().numpy(), db_ref) < 1e-4
    # ---- conv dgrad: equal to the undivided kernel
    wt = torch.from_numpy(np.ascontiguousarray(np.transpose(np.moveaxis(w, 1, -1), (4, 1, 2, 3, 0))).astype(np.float32)).cuda()
    gxh = host_empty(xh.numel())
    total = (xh.numel() + gch.numel()) * 4
    _chunked(lib, lambda wp, nb, inf: lib.lib.pooch_div_conv3d_dgrad(C.byref(d), ptr(gch), ptr(wt), ptr(gxh), wp, nb,
                                                                     sarr, inf), total)
    gxd = torch.full((xh.numel(),), float("nan"), device="cuda")
    lib.check(lib.lib.pooch_op_conv_dgrad(C.byref(d), ptr(gch.cuda()), ptr(wt), ptr(gxd), 0, None))
    torch.cuda.synchronize()
    assert torch.equal(gxh, gxd.cpu()), "divided dgrad differs from the undivided kernel"
    gc64 = ncdhw(gch.numpy().astype(np.float64).reshape(1, Do, Ho, Wo, K))
    assert rel(ncdhw(gxh.numpy().reshape(1, D, H, W, Cc)), L.conv3d_dgrad(gc64, w, x.shape, s, p)) < _tol_x3(K * k ** 3)
    # ---- conv wgrad: chunk partials summed in order
    dwd = torch.full_like(dw_dev, float("nan"))
    _chunked(lib, lambda wp, nb, inf: lib.lib.pooch_div_conv3d_wgrad(C.byref(d), ptr(xh), ptr(gch), ptr(dwd), wp, nb,
                                                                     sarr, inf),
             total + 4 * dw_dev.numel() + lib.lib.pooch_op_conv_wgrad_ws_bytes(C.byref(d)))
    torch.cuda.synchronize()
    gw_ref = L.conv3d_wgrad(x, gc64, w.shape, s, p)
    assert rel(np.moveaxis(dwd.cpu().numpy(), -1, 1), gw_ref) < _tol_x3(Do * Ho * Wo)


def test_divided_conv_infeasible_workspace():
    lib = _lib()
    d = lib.ConvDesc(1, 64, 64, 32, 32, 3, 3, 1, 1, 1, 8, 0, 0, 0)
    ws = torch.empty(1 << 16, dtype=torch.uint8, device="cuda")
    ss, sarr = _streams()
    x = host_empty(8 * 64 * 64 * 32)
    y = host_empty(8 * 64 * 64 * 32)
    w = torch.zeros(32 * 27 * 32, device="cuda")
    st = lib.lib.pooch_div_conv3d_fwd(C.byref(d), ptr(x), ptr(w), ptr(y), None, None, None, ptr(ws), 1 << 16, sarr,
                                      None)
    assert st == 2      # POOCH_EINFEASIBLE
