"""Pins for oracle/layers.py and oracle/nets.py math (C1): central finite
differences in fp64, closed forms, brute-force loops and library special
cases -- nothing here re-types the oracle's own formulas."""
import numpy as np
import pytest

from oracle import layers as L
from oracle import nets


def fd_grad(f, x, eps=1e-6):
    """Central finite differences of scalar f at x (all entries)."""
    g = np.zeros_like(x)
    it = np.nditer(x, flags=["multi_index"])
    for _ in it:
        idx = it.multi_index
        old = x[idx]
        x[idx] = old + eps
        fp = f()
        x[idx] = old - eps
        fm = f()
        x[idx] = old
        g[idx] = (fp - fm) / (2 * eps)
    return g


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def direct_conv(x, w, stride, pad):
    """Seven nested loops: the definition y[n,o,i,j] = sum x[..]*w[..]."""
    n, c, h, wd = x.shape
    o, _, r, s = w.shape
    ho = (h + 2 * pad - r) // stride + 1
    wo = (wd + 2 * pad - s) // stride + 1
    y = np.zeros((n, o, ho, wo))
    for a in range(n):
        for b in range(o):
            for i in range(ho):
                for j in range(wo):
                    acc = 0.0
                    for cc in range(c):
                        for u in range(r):
                            for v in range(s):
                                hi, wi = stride * i + u - pad, stride * j + v - pad
                                if 0 <= hi < h and 0 <= wi < wd:
                                    acc += x[a, cc, hi, wi] * w[b, cc, u, v]
                    y[a, b, i, j] = acc
    return y


@pytest.mark.parametrize("stride,pad,k", [(1, 1, 3), (2, 1, 3), (2, 0, 1), (1, 0, 1), (2, 3, 7)])
def test_conv_fwd_matches_direct_loops(stride, pad, k):
    g = np.random.default_rng(0)
    x = g.standard_normal((2, 3, 9, 8))
    w = g.standard_normal((4, 3, k, k))
    np.testing.assert_allclose(L.conv2d_fwd(x, w, stride, pad), direct_conv(x, w, stride, pad), rtol=1e-12, atol=1e-12)


def test_conv1x1_is_matmul():
    g = np.random.default_rng(1)
    x = g.standard_normal((2, 5, 4, 3))
    w = g.standard_normal((6, 5, 1, 1))
    ref = np.einsum("nchw,oc->nohw", x, w[:, :, 0, 0])
    ref2 = (x.transpose(0, 2, 3, 1).reshape(-1, 5) @ w[:, :, 0, 0].T).reshape(2, 4, 3, 6).transpose(0, 3, 1, 2)
    np.testing.assert_allclose(L.conv2d_fwd(x, w), ref2, rtol=1e-12)
    np.testing.assert_allclose(ref, ref2, rtol=1e-12)


@pytest.mark.parametrize("stride,pad,k", [(1, 1, 3), (2, 1, 3), (2, 0, 1)])
def test_conv_grads_fd(stride, pad, k):
    g = np.random.default_rng(2)
    x = g.standard_normal((2, 2, 6, 6))
    w = g.standard_normal((3, 2, k, k))
    y = L.conv2d_fwd(x, w, stride, pad)
    dy = g.standard_normal(y.shape)
    f = lambda: float((L.conv2d_fwd(x, w, stride, pad) * dy).sum())
    assert rel(L.conv2d_dgrad(dy, w, x.shape, stride, pad), fd_grad(f, x)) < 1e-7
    assert rel(L.conv2d_wgrad(x, dy, w.shape, stride, pad), fd_grad(f, w)) < 1e-7


def test_bn_fwd_stats_and_bwd_fd():
    g = np.random.default_rng(3)
    x = g.standard_normal((3, 2, 4, 4)) * 2 + 1
    gamma = g.uniform(0.5, 1.5, 2)
    beta = g.uniform(-1, 1, 2)
    y, cache = L.bn_fwd(x, gamma, beta)
    # normalised output has per-channel mean beta and biased variance ~gamma^2
    np.testing.assert_allclose(y.mean(axis=(0, 2, 3)), beta, atol=1e-12)
    np.testing.assert_allclose(y.var(axis=(0, 2, 3)), gamma ** 2 * x.var(axis=(0, 2, 3)) / (x.var(axis=(0, 2, 3)) + L.BN_EPS), rtol=1e-10)
    dy = g.standard_normal(y.shape)
    f = lambda: float((L.bn_fwd(x, gamma, beta)[0] * dy).sum())
    dx, dgm, dbt = L.bn_bwd(dy, cache, gamma)
    assert rel(dx, fd_grad(f, x)) < 1e-6
    assert rel(dgm, fd_grad(f, gamma)) < 1e-7
    assert rel(dbt, fd_grad(f, beta)) < 1e-7


def test_relu_and_pools_fd():
    g = np.random.default_rng(4)
    # distinct values, kept away from 0 and from pool ties
    x = g.permutation(np.linspace(-3, 3, 2 * 2 * 7 * 7)).reshape(2, 2, 7, 7)
    x[np.abs(x) < 1e-2] += 0.05
    y = L.relu_fwd(x)
    dy = g.standard_normal(y.shape)
    f = lambda: float((L.relu_fwd(x) * dy).sum())
    assert rel(L.relu_bwd(dy, y), fd_grad(f, x)) < 1e-8
    for k, s, p in [(3, 2, 1), (2, 2, 0)]:
        yp = L.maxpool_fwd(x, k, s, p)
        dyp = g.standard_normal(yp.shape)
        f = lambda: float((L.maxpool_fwd(x, k, s, p) * dyp).sum())
        assert rel(L.maxpool_bwd(dyp, x, k, s, p), fd_grad(f, x)) < 1e-8
    # avgpool is a mean
    np.testing.assert_allclose(L.avgpool_fwd(x), x.reshape(2, 2, -1).mean(-1))
    dya = g.standard_normal((2, 2))
    f = lambda: float((L.avgpool_fwd(x) * dya).sum())
    assert rel(L.avgpool_bwd(dya, x.shape), fd_grad(f, x)) < 1e-8


def test_maxpool_first_max_on_ties():
    x = np.zeros((1, 1, 2, 2))
    dx = L.maxpool_bwd(np.ones((1, 1, 1, 1)), x, 2, 2, 0)
    assert dx[0, 0, 0, 0] == 1 and dx.sum() == 1


def test_fc_and_ce():
    g = np.random.default_rng(5)
    x = g.standard_normal((4, 5))
    w = g.standard_normal((3, 5))
    b = g.standard_normal(3)
    t = np.array([0, 2, 1, 2])
    f = lambda: L.softmax_ce(L.fc_fwd(x, w, b), t)[0]
    loss, dz = L.softmax_ce(L.fc_fwd(x, w, b), t)
    # closed form: p - onehot over batch, rows sum to zero
    np.testing.assert_allclose(dz.sum(axis=1), 0, atol=1e-14)
    z = L.fc_fwd(x, w, b)
    p = np.exp(z) / np.exp(z).sum(1, keepdims=True)
    assert abs(loss - (-np.log(p[np.arange(4), t]).mean())) < 1e-12
    dx, dw, db = L.fc_bwd(dz, x, w)
    assert rel(dx, fd_grad(f, x)) < 1e-7
    assert rel(dw, fd_grad(f, w)) < 1e-7
    assert rel(db, fd_grad(f, b)) < 1e-7


def test_sgd_momentum_two_steps():
    w, v = np.array([1.0]), np.array([0.0])
    w, v = L.sgd_momentum(w, v, np.array([2.0]), 0.1)
    assert v[0] == 2.0 and abs(w[0] - 0.8) < 1e-15
    w, v = L.sgd_momentum(w, v, np.array([1.0]), 0.1)
    assert abs(v[0] - 2.8) < 1e-15 and abs(w[0] - 0.52) < 1e-15


def _micro_resnet():
    """Small net with every task kind of ResNet-50 (both tail variants)."""
    net = nets.Net("micro", (3, 8, 8), 4)
    T = nets.Task
    c = net.add(T("c0", "conv", [-1], (4, 4, 4), 2, 1, 3, 3))
    x = net.add(T("b0", "bnrelu", [c], (4, 4, 4)))
    x = net.add(T("mp", "maxpool", [x], (4, 2, 2), 2, 1, 3))
    c1 = net.add(T("l.conv1", "conv", [x], (2, 2, 2), 1, 0, 1, 4))
    y1 = net.add(T("l.bn1", "bnrelu", [c1], (2, 2, 2)))
    c3 = net.add(T("l.conv3", "conv", [y1], (6, 1, 1), 2, 1, 3, 2))
    pj = net.add(T("l.downsample", "conv", [x], (6, 1, 1), 2, 0, 1, 4))
    x = net.add(T("l.tail", "tail_proj", [c3, pj], (6, 1, 1)))
    c4 = net.add(T("m.conv1", "conv", [x], (6, 1, 1), 1, 0, 1, 6))
    x = net.add(T("m.tail", "tail_id", [c4, x], (6, 1, 1)))
    a = net.add(T("avgpool", "avgpool", [x], (6, 1, 1)))
    net.add(T("fc", "fc_ce", [a], (4, 1, 1), cin=6))
    return net


def test_net_forward_backward_fd():
    net = _micro_resnet()
    params = {k: v.astype(np.float64) for k, v in nets.init_params(net, seed=7, bn_random=True).items()}
    g = np.random.default_rng(8)
    x = g.standard_normal((3, 8, 8, 3))
    t = np.array([1, 3, 0])
    loss, grads, _ = nets.forward_backward(net, params, x, t)
    for name in ["c0.w", "l.conv3.w", "l.downsample.w", "m.conv1.w", "b0.gamma", "l.tail.betap",
                 "m.tail.gamma3", "fc.w", "fc.b"]:
        f = lambda: nets.forward_backward(net, params, x, t)[0]
        assert rel(grads[name], fd_grad(f, params[name])) < 1e-5, name


def test_tiny_cnn_fd_spot():
    net = nets.tiny_cnn(width=4, in_hw=6)
    params = {k: v.astype(np.float64) for k, v in nets.init_params(net, seed=3, bn_random=True).items()}
    x = np.random.default_rng(9).standard_normal((2, 6, 6, 3))
    t = np.array([1, 7])
    loss, grads, _ = nets.forward_backward(net, params, x, t)
    for name in ["conv0.w", "bn2.gamma", "conv3.w", "fc.w"]:
        f = lambda: nets.forward_backward(net, params, x, t)[0]
        assert rel(grads[name], fd_grad(f, params[name])) < 1e-5, name


def test_tf32_operand_rounding_bits():
    """tf32() keeps sign, exponent and the top 10 mantissa bits of the fp32 value."""
    x = np.array([1.0, 1.0 + 2.0 ** -10, 1.0 + 2.0 ** -11, -3.0000001, 2.0 ** -126, 65504.123, 0.0])
    q = L.tf32(x)
    u = q.astype(np.float32).view(np.uint32)
    assert np.all(u & 0x1FFF == 0)
    assert q[0] == 1.0 and q[1] == 1.0 + 2.0 ** -10 and q[2] == 1.0      # truncation, not rounding
    assert np.all(np.abs(q) <= np.abs(x.astype(np.float32)))              # toward zero
    assert np.array_equal(L.tf32(q), q)                                   # idempotent
    r = np.random.default_rng(0).standard_normal(10000)
    rel = np.abs(L.tf32(r) - r) / np.abs(r)
    assert rel.max() < 2.0 ** -10 + 1e-7
