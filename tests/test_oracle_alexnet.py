"""Pins for the oracle's AlexNet workload: the LRN layer against a
brute-force loop and a closed form, every new adjoint against central finite differences, the
counter-based dropout generator against MurmurHash3's published finaliser value and its
statistics, and the census against AlexNet's well-known parameter count."""
import numpy as np
import pytest

import synthdata
from oracle import layers as L
from oracle import nets


def test_fmix32_is_murmur3_finaliser():
    # MurmurHash3 fmix32: fmix32(0) = 0 and fmix32(1) = 0x514E28B7 (the reference implementation)
    assert int(L._fmix32(np.uint32(0))) == 0
    assert int(L._fmix32(np.uint32(1))) == 0x514E28B7


def test_dropout_mask_statistics_and_determinism():
    m = L.dropout_keep((1000, 1000), 0.5, 7, 3, 11)
    assert abs(m.mean() - 0.5) < 2e-3                                   # Bernoulli(0.5), n = 1e6
    assert np.array_equal(m, L.dropout_keep((1000, 1000), 0.5, 7, 3, 11))   # a pure function
    other = L.dropout_keep((1000, 1000), 0.5, 7, 4, 11)                 # next step: a new mask
    assert abs((m == other).mean() - 0.5) < 3e-3                        # independent of the last
    assert L.dropout_keep((10, 10), 0.0, 1, 2, 3).all()
    assert abs(L.dropout_keep((1000, 1000), 0.25, 0, 0, 0).mean() - 0.75) < 2e-3


def _lrn_loops(x, n=5, k=2.0, alpha=1e-4, beta=0.75):
    """LRN written element by element (independent of lrn_fwd's vectorised windows)."""
    N, C, H, W = x.shape
    y = np.zeros_like(x)
    for a in range(N):
        for c in range(C):
            for i in range(H):
                for j in range(W):
                    s = 0.0
                    for cc in range(C):
                        if abs(cc - c) <= n // 2:
                            s += x[a, cc, i, j] ** 2
                    y[a, c, i, j] = x[a, c, i, j] / (k + alpha / n * s) ** beta
    return y


def test_lrn_against_loops_and_closed_form():
    g = synthdata.rng(1)
    x = g.standard_normal((2, 9, 3, 2)) * 20.0          # large enough that the window term matters
    np.testing.assert_allclose(L.lrn_fwd(x)[0], _lrn_loops(x), rtol=1e-13, atol=0)
    # a single non-zero channel a: y = a / (2 + 1e-4 / 5 * a^2)^0.75, its neighbours stay 0
    x1 = np.zeros((1, 7, 1, 1))
    x1[0, 3] = 30.0
    y1 = L.lrn_fwd(x1)[0]
    assert y1[0, 3, 0, 0] == pytest.approx(30.0 / (2.0 + 1e-4 / 5 * 900.0) ** 0.75, rel=1e-15)
    assert np.count_nonzero(y1) == 1


def _fd(f, x, idx, h=1e-6):
    xp, xm = x.copy(), x.copy()
    xp[idx] += h
    xm[idx] -= h
    return (f(xp) - f(xm)) / (2 * h)


def test_lrn_backward_finite_differences():
    g = synthdata.rng(2)
    x = g.standard_normal((2, 11, 3, 3)) * 30.0
    dy = g.standard_normal(x.shape)
    dx = L.lrn_bwd(dy, x)
    for _ in range(25):
        idx = tuple(int(g.integers(0, s)) for s in x.shape)
        num = _fd(lambda v: float((L.lrn_fwd(v)[0] * dy).sum()), x, idx, 1e-5)
        assert dx[idx] == pytest.approx(num, rel=1e-6, abs=1e-9)


def test_conv_bias_relu_and_fc_dropout_finite_differences():
    g = synthdata.rng(3)
    x = g.standard_normal((2, 3, 9, 9))
    w = g.standard_normal((4, 3, 3, 3)) * 0.3
    b = g.standard_normal(4) * 0.1
    y = L.relu_fwd(L.conv2d_bias_fwd(x, w, b, 2, 1))
    dy = g.standard_normal(y.shape)
    dz = L.relu_bwd(dy, y)
    db = dz.sum(axis=(0, 2, 3))
    for c in range(4):
        num = _fd(lambda v: float((L.relu_fwd(L.conv2d_bias_fwd(x, w, v, 2, 1)) * dy).sum()), b, (c,))
        assert db[c] == pytest.approx(num, rel=1e-6, abs=1e-9)
    # FC + ReLU + inverted dropout with a fixed mask
    xf = g.standard_normal((5, 12))
    wf = g.standard_normal((8, 12)) * 0.3
    bf = g.standard_normal(8) * 0.1
    keep = L.dropout_keep((5, 8), 0.5, 1, 2, 3)
    yf, z = L.fc_relu_dropout_fwd(xf, wf, bf, keep, 0.5)
    dyf = g.standard_normal(yf.shape)
    dx, dw, dbf = L.fc_relu_dropout_bwd(dyf, xf, wf, z, keep, 0.5)
    loss = lambda xx, ww, bb: float((L.fc_relu_dropout_fwd(xx, ww, bb, keep, 0.5)[0] * dyf).sum())  # noqa: E731
    for _ in range(10):
        i, j = int(g.integers(0, 5)), int(g.integers(0, 12))
        assert dx[i, j] == pytest.approx(_fd(lambda v: loss(v, wf, bf), xf, (i, j)), rel=1e-6, abs=1e-9)
        o = int(g.integers(0, 8))
        assert dw[o, j] == pytest.approx(_fd(lambda v: loss(xf, v, bf), wf, (o, j)), rel=1e-6, abs=1e-9)
        assert dbf[o] == pytest.approx(_fd(lambda v: loss(xf, wf, v), bf, (o,)), rel=1e-6, abs=1e-9)
    assert np.all(yf[~keep] == 0) and np.allclose(yf[keep], 2.0 * np.maximum(z[keep], 0))


def test_alexnet_census():
    net = nets.alexnet()
    shapes = nets.param_shapes(net)
    # the single-tower (ungrouped) AlexNet: 62,378,344 parameters (conv 3,747,200 + fc 58,631,144)
    assert sum(int(np.prod(s)) for s in shapes.values()) == 62378344
    cen = nets.census(net, 1)
    assert len(cen) == 13
    # per-image map bytes (fp32), by hand: 96x55x55 (x2: ReLU, LRN), 96x27x27, 256x27x27 (x2),
    # 256x13x13, 384x13x13 (x2), 256x13x13, 256x6x6, 4096 (x2), 1000
    expect = [96 * 55 * 55] * 2 + [96 * 27 * 27] + [256 * 27 * 27] * 2 + [256 * 13 * 13] + [384 * 169] * 2 + \
        [256 * 169, 256 * 36, 4096, 4096, 1000]
    assert [b for _, b in cen] == [4 * e for e in expect]
    assert sum(b for _, b in cen) == 5035040


def test_micro_alexnet_whole_net_finite_differences():
    """Whole-step gradients of the 67x67 AlexNet (every task kind, dropout masks fixed by the
    counter-based generator) against central differences of the loss."""
    net = nets.alexnet(in_hw=67)
    params = nets.init_params(net, seed=2)
    for k in params:
        if k.endswith(".b"):
            params[k] = synthdata.rng(5).uniform(-0.05, 0.05, params[k].shape).astype(np.float32)
    x = synthdata.images(2, 67, 67, 3, seed=0)
    t = synthdata.labels(2, 1000, seed=1)
    loss, grads, _ = nets.forward_backward(net, params, x, t, rng=(3, 1))
    g = synthdata.rng(6)
    P64 = {k: np.asarray(v, np.float64) for k, v in params.items()}
    for name in ("conv1.w", "conv1.b", "conv2.w", "conv4.b", "fc6.w", "fc7.b", "fc8.w"):
        for _ in range(2):
            idx = tuple(int(g.integers(0, s)) for s in P64[name].shape)
            if name == "fc6.w":   # a weight with a live (kept, positive) unit
                idx = (int(np.argmax(np.abs(grads[name]).sum(axis=1))), idx[1])
            h = 1e-4 * max(1.0, abs(P64[name][idx]))

            def f(v):
                q = dict(P64)
                q[name] = v
                return nets.forward_backward(net, q, x, t, rng=(3, 1))[0]
            num = _fd(f, P64[name], idx, h)
            assert grads[name][idx] == pytest.approx(num, rel=2e-4, abs=1e-7), (name, idx)


def test_decisions_mode():
    """oracle.nets ``decisions``: discrete choices taken from given tensors (the GPU's maps).
    (a) The pool helpers reproduce the pinned max-pool definitions when the winners come from the
    same tensor; (b) a hand example where the given tensor picks another winner; (c) feeding the
    oracle its own outputs as decisions changes nothing (tiny CNN and 67^2 AlexNet)."""
    g = synthdata.rng(12)
    x = g.standard_normal((2, 3, 7, 7))
    for k, s, p in ((3, 2, 1), (3, 2, 0), (2, 2, 0)):
        arg = L.maxpool_argmax(x, k, s, p)
        y = L.maxpool_fwd_at(x, arg, k, s, p)
        assert np.array_equal(y, L.maxpool_fwd(x, k, s, p))
        dy = g.standard_normal(y.shape)
        assert np.array_equal(L.maxpool_bwd_at(dy, x.shape, arg, k, s, p), L.maxpool_bwd(dy, x, k, s, p))
    # 2x2 window [[1, 2], [3, 0]] whose winner is decided by [[5, 0], [0, 0]]: y = 1, dx at (0, 0)
    xx = np.array([[[[1.0, 2.0], [3.0, 0.0]]]])
    arg = L.maxpool_argmax(np.array([[[[5.0, 0.0], [0.0, 0.0]]]]), 2, 2, 0)
    assert L.maxpool_fwd_at(xx, arg, 2, 2, 0)[0, 0, 0, 0] == 1.0
    assert np.array_equal(L.maxpool_bwd_at(np.array([[[[7.0]]]]), xx.shape, arg, 2, 2, 0),
                          np.array([[[[7.0, 0.0], [0.0, 0.0]]]]))
    for net, hw, cls in ((nets.tiny_cnn(), 32, 10), (nets.alexnet(in_hw=67), 67, 1000)):
        params = nets.init_params(net, seed=2, bn_random=True)
        xi = synthdata.images(2, hw, hw, 3, seed=0)
        t = synthdata.labels(2, cls, seed=1)
        l0, g0, outs = nets.forward_backward(net, params, xi, t, rng=(1, 2))
        dec = {}
        for i, tk in enumerate(net.tasks):
            if tk.kind in ("bnrelu", "tail_proj", "tail_id", "conv_relu", "fc_relu_drop"):
                dec[i] = outs[i]
            elif tk.kind == "maxpool":
                dec[i] = outs[tk.inputs[0]]
        l1, g1, _ = nets.forward_backward(net, params, xi, t, rng=(1, 2), decisions=dec)
        assert l1 == pytest.approx(l0, rel=1e-12)
        for k in g0:
            np.testing.assert_allclose(g1[k], g0[k], rtol=1e-10, atol=1e-14)
