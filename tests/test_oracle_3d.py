"""Pins for the 3D U-Net part of the oracle (BASELINE.json config 4): conv3d,
transposed conv3d (k2 s2), 3D max-pool, N-d BatchNorm, per-voxel softmax-CE and
the U-Net census. Each check is against something other than the oracle's own
formula: direct nested loops, finite differences, the conv2d special case, the
adjoint identity transposed-conv = conv-dgrad, or the SURVEY 8(d) census."""
import itertools

import numpy as np
import pytest

from oracle import layers as L
from oracle import nets

from test_oracle_layers import fd_grad, rel


def direct_conv3d(x, w, stride, pad):
    """The definition y[n,o,a,i,j] = sum_{c,u,v,t} x[..] w[..], as plain loops."""
    n, c, d, h, wd = x.shape
    o, _, k, _, _ = w.shape
    do, ho, wo = ((e + 2 * pad - k) // stride + 1 for e in (d, h, wd))
    y = np.zeros((n, o, do, ho, wo))
    for b, oo, a, i, j in itertools.product(range(n), range(o), range(do), range(ho), range(wo)):
        acc = 0.0
        for cc, u, v, t in itertools.product(range(c), range(k), range(k), range(k)):
            zi, hi, wi = stride * a + u - pad, stride * i + v - pad, stride * j + t - pad
            if 0 <= zi < d and 0 <= hi < h and 0 <= wi < wd:
                acc += x[b, cc, zi, hi, wi] * w[oo, cc, u, v, t]
        y[b, oo, a, i, j] = acc
    return y


@pytest.mark.parametrize("stride,pad,k", [(1, 1, 3), (2, 0, 2), (1, 0, 1), (2, 1, 3)])
def test_conv3d_fwd_matches_direct_loops(stride, pad, k):
    g = np.random.default_rng(1)
    x = g.standard_normal((1, 2, 5, 4, 6))
    w = g.standard_normal((3, 2, k, k, k))
    np.testing.assert_allclose(L.conv3d_fwd(x, w, stride, pad), direct_conv3d(x, w, stride, pad),
                               rtol=1e-12, atol=1e-12)


def test_conv3d_reduces_to_conv2d():
    """A depth-1 volume with only the centre depth tap of a 3^3 kernel is a 2D conv."""
    g = np.random.default_rng(2)
    x = g.standard_normal((2, 3, 1, 7, 6))
    w2 = g.standard_normal((4, 3, 3, 3))
    w3 = np.zeros((4, 3, 3, 3, 3))
    w3[:, :, 1] = w2
    y3 = L.conv3d_fwd(x, w3, 1, 1)
    np.testing.assert_allclose(y3[:, :, 0], L.conv2d_fwd(x[:, :, 0], w2, 1, 1), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("stride,pad,k", [(1, 1, 3), (2, 0, 2)])
def test_conv3d_grads_fd(stride, pad, k):
    g = np.random.default_rng(3)
    x = g.standard_normal((1, 2, 4, 4, 3))
    w = g.standard_normal((2, 2, k, k, k))
    dy = g.standard_normal(L.conv3d_fwd(x, w, stride, pad).shape)
    f = lambda: float((L.conv3d_fwd(x, w, stride, pad) * dy).sum())
    assert rel(L.conv3d_dgrad(dy, w, x.shape, stride, pad), fd_grad(f, x)) < 1e-7
    assert rel(L.conv3d_wgrad(x, dy, w.shape, stride, pad), fd_grad(f, w)) < 1e-7


def test_upconv_is_the_adjoint_of_a_k2s2_conv():
    """A transposed convolution is the input-gradient of the convolution with the same
    weights: upconv3d(x, w) = conv3d_dgrad(x, w, stride 2, pad 0)."""
    g = np.random.default_rng(4)
    x = g.standard_normal((2, 3, 2, 3, 2))
    w = g.standard_normal((3, 5, 2, 2, 2))                # [Cin, Cout, 2, 2, 2]
    y = L.upconv3d_fwd(x, w)
    assert y.shape == (2, 5, 4, 6, 4)
    np.testing.assert_allclose(y, L.conv3d_dgrad(x, w, (2, 5, 4, 6, 4), 2, 0), rtol=1e-12, atol=1e-12)
    # every output voxel receives exactly one tap: spot-check one voxel by hand
    n, o, a, i, j = 1, 4, 3, 5, 2
    ref = sum(x[n, c, a // 2, i // 2, j // 2] * w[c, o, a % 2, i % 2, j % 2] for c in range(3))
    assert abs(y[n, o, a, i, j] - ref) < 1e-12


def test_upconv_grads_fd():
    g = np.random.default_rng(5)
    x = g.standard_normal((1, 2, 2, 2, 3))
    w = g.standard_normal((2, 3, 2, 2, 2))
    dy = g.standard_normal((1, 3, 4, 4, 6))
    f = lambda: float((L.upconv3d_fwd(x, w) * dy).sum())
    dx, dw = L.upconv3d_bwd(dy, x, w)
    assert rel(dx, fd_grad(f, x)) < 1e-7
    assert rel(dw, fd_grad(f, w)) < 1e-7


def test_maxpool3d_windows_and_grad():
    g = np.random.default_rng(6)
    x = g.standard_normal((2, 3, 4, 6, 4))
    y = L.maxpool3d_fwd(x)
    for b, c, a, i, j in itertools.product(range(2), range(3), range(2), range(3), range(2)):
        assert y[b, c, a, i, j] == x[b, c, 2 * a:2 * a + 2, 2 * i:2 * i + 2, 2 * j:2 * j + 2].max()
    dy = g.standard_normal(y.shape)
    f = lambda: float((L.maxpool3d_fwd(x) * dy).sum())
    assert rel(L.maxpool3d_bwd(dy, x), fd_grad(f, x)) < 1e-7


def test_maxpool3d_first_max_on_ties():
    x = np.zeros((1, 1, 2, 2, 2))
    dx = L.maxpool3d_bwd(np.ones((1, 1, 1, 1, 1)), x)
    assert dx[0, 0, 0, 0, 0] == 1.0 and dx.sum() == 1.0


def test_bn_3d_equals_2d_on_a_reshaped_volume():
    g = np.random.default_rng(7)
    x = g.standard_normal((2, 3, 4, 5, 2))
    gam, bet = g.uniform(0.5, 1.5, 3), g.uniform(-1, 1, 3)
    y3, c3 = L.bn_fwd(x, gam, bet)
    y2, c2 = L.bn_fwd(x.reshape(2, 3, 20, 2), gam, bet)
    np.testing.assert_allclose(y3.reshape(2, 3, 20, 2), y2, rtol=1e-12, atol=1e-12)
    dy = g.standard_normal(x.shape)
    d3 = L.bn_bwd(dy, c3, gam)
    d2 = L.bn_bwd(dy.reshape(2, 3, 20, 2), c2, gam)
    np.testing.assert_allclose(d3[0].reshape(2, 3, 20, 2), d2[0], rtol=1e-12, atol=1e-12)


def _micro_unet():
    """Every 3D task kind, tiny: encoder level, pool, bottleneck conv, upconv, two-input
    (concatenating) conv, head with voxel CE."""
    net = nets.Net("micro3d", (1, 4, 4, 4), 3)
    T = nets.Task
    c0 = net.add(T("e.conv", "conv", [-1], (2, 4, 4, 4), 1, 1, 3, 1))
    y0 = net.add(T("e.bn", "bnrelu", [c0], (2, 4, 4, 4)))
    p = net.add(T("pool", "maxpool", [y0], (2, 2, 2, 2), 2, 0, 2))
    c1 = net.add(T("m.conv", "conv", [p], (3, 2, 2, 2), 1, 1, 3, 2))
    y1 = net.add(T("m.bn", "bnrelu", [c1], (3, 2, 2, 2)))
    u = net.add(T("up", "upconv", [y1], (2, 4, 4, 4), 2, 0, 2, 3))
    c2 = net.add(T("d.conv", "conv", [u, y0], (2, 4, 4, 4), 1, 1, 3, 4))
    y2 = net.add(T("d.bn", "bnrelu", [c2], (2, 4, 4, 4)))
    net.add(T("head", "head_ce", [y2], (3, 4, 4, 4), cin=2))
    return net


def test_micro_unet_forward_backward_fd():
    net = _micro_unet()
    params = {k: v.astype(np.float64) for k, v in nets.init_params(net, seed=11, bn_random=True).items()}
    g = np.random.default_rng(12)
    x = g.standard_normal((2, 4, 4, 4, 1))
    t = g.integers(0, 3, (2, 4, 4, 4))
    loss, grads, outs = nets.forward_backward(net, params, x, t)
    assert outs[-1].shape == (2, 3, 4, 4, 4)
    for name in ["e.conv.w", "m.conv.w", "up.w", "d.conv.w", "e.bn.gamma", "d.bn.beta", "head.w", "head.b"]:
        f = lambda: nets.forward_backward(net, params, x, t)[0]
        assert rel(grads[name], fd_grad(f, params[name])) < 1e-5, name


def test_head_ce_is_the_mean_over_voxels():
    """The per-voxel head equals a batch of independent FC + CE rows (one per voxel)."""
    net = nets.Net("h", (2, 2, 2, 2), 3)
    net.add(nets.Task("head", "head_ce", [-1], (3, 2, 2, 2), cin=2))
    g = np.random.default_rng(13)
    p = {"head.w": g.standard_normal((3, 2)), "head.b": g.standard_normal(3)}
    x = g.standard_normal((1, 2, 2, 2, 2))
    t = g.integers(0, 3, (1, 2, 2, 2))
    loss, _, _ = nets.forward_backward(net, p, x, t)
    z = x.reshape(8, 2) @ p["head.w"].T + p["head.b"]
    lp = z - np.log(np.exp(z).sum(1, keepdims=True))
    assert abs(loss - (-lp[np.arange(8), t.reshape(-1)].mean())) < 1e-12


def test_unet3d_census_matches_survey():
    """45 maps, 207.2 GB at 256^3 (batch 1), largest map 17.2 GB,
    386.6 M parameters; decoder first convs read 27 x 512 = 13,824 K at level 1."""
    net = nets.unet3d()
    cen = nets.census(net, 1)
    assert len(cen) == 45
    tot = sum(b for _, b in cen)
    assert abs(tot / 1e9 - 207.2) < 0.05
    assert abs(max(b for _, b in cen) / 1e9 - 17.18) < 0.01
    nparam = sum(int(np.prod(s)) for s in nets.param_shapes(net).values())
    assert abs(nparam / 1e6 - 386.6) < 0.1
    d1 = [t for t in net.tasks if t.name == "dec1.conv1"][0]
    assert d1.cin * 27 == 13824 and len(d1.inputs) == 2
