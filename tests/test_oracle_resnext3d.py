"""Pins for the ResNeXt-101 (3D) part of the oracle: grouped
3D convolution with a per-axis stride, the padded 3^3 / 2 max-pool, the N-d global average pool
and the network. Each check is against something other than the oracle's own formula: direct
nested loops of the definition, the groups = 1 special case (the pinned conv3d), the adjoint
identities, finite differences of the whole network, and counts derived by hand."""
import itertools

import numpy as np
import pytest

from oracle import layers as L
from oracle import nets

from test_oracle_layers import fd_grad, rel


def direct_gconv3d(x, w, s3, pad, groups):
    """y[n, g*Og+o, a, i, j] = sum_{c < Cg, u, v, t} x[n, g*Cg+c, sd*a+u-p, sh*i+v-p, sw*j+t-p]
    * w[g*Og+o, c, u, v, t], as plain loops over every index."""
    n, C, d, h, wd = x.shape
    O, cg, k, _, _ = w.shape
    og = O // groups
    sd, sh, sw = s3
    do, ho, wo = (d + 2 * pad - k) // sd + 1, (h + 2 * pad - k) // sh + 1, (wd + 2 * pad - k) // sw + 1
    y = np.zeros((n, O, do, ho, wo))
    for b, oo, a, i, j in itertools.product(range(n), range(O), range(do), range(ho), range(wo)):
        g = oo // og
        acc = 0.0
        for c, u, v, t in itertools.product(range(cg), range(k), range(k), range(k)):
            zi, hi, wi = sd * a + u - pad, sh * i + v - pad, sw * j + t - pad
            if 0 <= zi < d and 0 <= hi < h and 0 <= wi < wd:
                acc += x[b, g * cg + c, zi, hi, wi] * w[oo, c, u, v, t]
        y[b, oo, a, i, j] = acc
    return y


@pytest.mark.parametrize("s3,pad,k,groups,C,O", [((1, 1, 1), 1, 3, 2, 4, 6), ((2, 2, 2), 1, 3, 4, 8, 8),
                                                  ((1, 2, 2), 3, 7, 1, 3, 2), ((2, 2, 2), 0, 1, 1, 4, 3),
                                                  ((1, 1, 1), 1, 3, 4, 4, 4)])
def test_gconv3d_fwd_matches_direct_loops(s3, pad, k, groups, C, O):
    """Includes depthwise (groups = C = O), the (1, 2, 2)-strided 7^3 stem and a strided 1^3."""
    g = np.random.default_rng(1)
    x = g.standard_normal((1, C, 5, 6, 7))
    w = g.standard_normal((O, C // groups, k, k, k))
    np.testing.assert_allclose(L.gconv3d_fwd(x, w, s3, pad, groups), direct_gconv3d(x, w, s3, pad, groups),
                               rtol=1e-12, atol=1e-12)


def test_gconv3d_groups1_is_conv3d():
    g = np.random.default_rng(2)
    x = g.standard_normal((2, 3, 5, 4, 6))
    w = g.standard_normal((4, 3, 3, 3, 3))
    np.testing.assert_allclose(L.gconv3d_fwd(x, w, 2, 1, 1), L.conv3d_fwd(x, w, 2, 1), rtol=1e-12, atol=1e-12)
    dy = g.standard_normal(L.conv3d_fwd(x, w, 2, 1).shape)
    np.testing.assert_allclose(L.gconv3d_dgrad(dy, w, x.shape, 2, 1, 1), L.conv3d_dgrad(dy, w, x.shape, 2, 1),
                               rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(L.gconv3d_wgrad(x, dy, w.shape, 2, 1, 1), L.conv3d_wgrad(x, dy, w.shape, 2, 1),
                               rtol=1e-12, atol=1e-12)


def test_gconv3d_is_block_diagonal():
    """A grouped conv equals the dense conv whose weight is zero outside the group blocks."""
    g = np.random.default_rng(3)
    G, cg, og = 4, 2, 3
    x = g.standard_normal((1, G * cg, 4, 5, 4))
    w = g.standard_normal((G * og, cg, 3, 3, 3))
    dense = np.zeros((G * og, G * cg, 3, 3, 3))
    for q in range(G):
        dense[q * og:(q + 1) * og, q * cg:(q + 1) * cg] = w[q * og:(q + 1) * og]
    np.testing.assert_allclose(L.gconv3d_fwd(x, w, (1, 2, 2), 1, G), L.gconv3d_fwd(x, dense, (1, 2, 2), 1, 1),
                               rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("s3,groups", [((1, 1, 1), 2), ((2, 2, 2), 4), ((1, 2, 2), 1)])
def test_gconv3d_grads_fd(s3, groups):
    g = np.random.default_rng(4)
    x = g.standard_normal((1, 4, 4, 5, 4))
    w = g.standard_normal((4, 4 // groups, 3, 3, 3))
    dy = g.standard_normal(L.gconv3d_fwd(x, w, s3, 1, groups).shape)
    f = lambda: float((L.gconv3d_fwd(x, w, s3, 1, groups) * dy).sum())
    assert rel(L.gconv3d_dgrad(dy, w, x.shape, s3, 1, groups), fd_grad(f, x)) < 1e-7
    assert rel(L.gconv3d_wgrad(x, dy, w.shape, s3, 1, groups), fd_grad(f, w)) < 1e-7


def test_maxpool3d_padded_windows_and_grad():
    """3^3 / 2, pad 1 (ResNeXt-101 (3D)): every output is the max of its clipped window; the
    gradient is the finite difference (ties have probability 0 for Gaussian input)."""
    g = np.random.default_rng(5)
    x = g.standard_normal((1, 2, 5, 6, 4))
    y = L.maxpool3d_fwd(x, 3, 2, 1)
    assert y.shape == (1, 2, 3, 3, 2)
    for b, c, a, i, j in itertools.product(range(1), range(2), range(3), range(3), range(2)):
        win = x[b, c, max(2 * a - 1, 0):2 * a + 2, max(2 * i - 1, 0):2 * i + 2, max(2 * j - 1, 0):2 * j + 2]
        assert y[b, c, a, i, j] == win.max()
    dy = g.standard_normal(y.shape)
    f = lambda: float((L.maxpool3d_fwd(x, 3, 2, 1) * dy).sum())
    assert rel(L.maxpool3d_bwd(dy, x, 3, 2, 1), fd_grad(f, x)) < 1e-7
    arg = L.maxpool3d_argmax(x, 3, 2, 1)
    np.testing.assert_array_equal(L.maxpool3d_fwd_at(x, arg, 3, 2, 1), y)
    np.testing.assert_array_equal(L.maxpool3d_bwd_at(dy, x.shape, arg, 3, 2, 1), L.maxpool3d_bwd(dy, x, 3, 2, 1))


def test_maxpool3d_padded_first_max_on_ties():
    """Overlapping windows (stride 2 < k 3): a tie inside a window goes to its first position;
    the -inf padding never wins."""
    x = np.zeros((1, 1, 3, 3, 3))
    dx = L.maxpool3d_bwd(np.ones((1, 1, 2, 2, 2)), x, 3, 2, 1)
    # window (0,0,0) covers input [0:2]^3: first max at input (0,0,0); window (1,1,1) covers
    # [1:3]^3: first at (1,1,1); windows mixing 0/1 starts take (0|1, 0|1, 0|1) accordingly
    assert dx.sum() == 8.0 and dx[0, 0, 0, 0, 0] == 1.0 and dx[0, 0, 1, 1, 1] == 1.0


def test_avgpool_nd_is_the_mean():
    g = np.random.default_rng(6)
    x = g.standard_normal((2, 3, 2, 3, 4))
    np.testing.assert_allclose(L.avgpool_fwd(x), x.reshape(2, 3, -1).mean(-1), rtol=1e-13)
    dy = g.standard_normal((2, 3))
    dx = L.avgpool_bwd(dy, x.shape)
    f = lambda: float((L.avgpool_fwd(x) * dy).sum())
    assert rel(dx, fd_grad(f, x)) < 1e-8


def _micro():
    """Every ResNeXt-3D task kind at FD size: (1, 2, 2)-strided 7^3 stem, padded pool, grouped
    3^3 convs (stride 1 and 2), projection and identity tails, avgpool + FC."""
    return nets.resnext3d((4, 8, 8), classes=3, cardinality=2, widths=(4, 4), blocks=[2, 1], stem=4)


def test_micro_resnext3d_forward_backward_fd():
    net = _micro()
    kinds = {t.kind for t in net.tasks}
    assert kinds == {"conv", "bnrelu", "maxpool", "tail_proj", "tail_id", "avgpool", "fc_ce"}
    assert any(t.groups == 2 and t.stride == 2 for t in net.tasks)
    params = {k: v.astype(np.float64) for k, v in nets.init_params(net, seed=21, bn_random=True).items()}
    g = np.random.default_rng(22)
    x = g.standard_normal((1, 4, 8, 8, 3))
    t = np.array([1])
    loss, grads, outs = nets.forward_backward(net, params, x, t)
    assert outs[0].shape == (1, 4, 4, 4, 4)         # stem: depth stride 1, H / W stride 2
    f = lambda: nets.forward_backward(net, params, x, t)[0]
    for name in ["conv1.w", "layer1.0.conv2.w", "layer2.0.conv2.w", "layer1.0.downsample.w", "layer1.1.conv1.w",
                 "bn1.gamma", "layer2.0.tail.gammap", "layer1.1.tail.beta3", "fc.w"]:
        # directional derivatives along 3 random unit directions (a full FD of the 4,116-entry
        # stem weight takes minutes): f(p + e v) - f(p - e v) / 2e = <grad, v>
        p0 = params[name].copy()
        for k in range(3):
            v = g.standard_normal(p0.shape)
            v /= np.linalg.norm(v)
            params[name] = p0 + 1e-6 * v
            fp = f()
            params[name] = p0 - 1e-6 * v
            fm = f()
            params[name] = p0
            fd = (fp - fm) / 2e-6
            an = float((grads[name] * v).sum())
            assert abs(fd - an) <= 1e-5 * max(abs(an), 1e-3 * np.linalg.norm(grads[name])), (name, fd, an)


def test_resnext101_3d_census():
    """Counted by hand from the architecture: stem conv + BN-ReLU + pool (3 maps), 33 blocks x
    (conv1, bn1, conv2, bn2, conv3, tail) + 4 projections, avgpool, fc = 3 + 198 + 4 + 2 = 207
    maps. Parameters: stem 64*3*343 + BN 2*64; block of width m, input c_in, output 2m:
    m*c_in + 2m (BN) + m*(m/32)*27 + 2m + 2m*m + 2*2m (tail BN) [+ 2m*c_in + 2*2m projection];
    FC 2048*400 + 400."""
    net = nets.resnext3d()
    assert len(nets.census(net, 1)) == 207
    total = 64 * 3 * 343 + 2 * 64
    cin = 64
    for nb, m in zip([3, 4, 23, 3], [128, 256, 512, 1024]):
        for b in range(nb):
            total += m * cin + 2 * m + m * (m // 32) * 27 + 2 * m + 2 * m * m + 2 * 2 * m
            if b == 0:
                total += 2 * m * cin + 2 * 2 * m
            cin = 2 * m
    total += 2048 * 400 + 400
    assert sum(int(np.prod(s)) for s in nets.param_shapes(net).values()) == total
    # the first grouped conv has 32 groups of 4 channels; the stride-2 ones halve D, H and W
    c2 = [t for t in net.tasks if t.name == "layer2.0.conv2"][0]
    assert c2.groups == 32 and c2.cin // c2.groups == 8 and c2.stride == 2
    # shapes at Hara et al.'s 16 x 112 x 112 clip: stem (16, 56, 56), pool (8, 28, 28),
    # stages (8, 28, 28) / (4, 14, 14) / (2, 7, 7) / (1, 4, 4)
    shp = {t.name: t.out_chw for t in net.tasks}
    assert shp["conv1"] == (64, 16, 56, 56) and shp["maxpool"] == (64, 8, 28, 28)
    assert shp["layer1.2.tail"] == (256, 8, 28, 28) and shp["layer4.2.tail"] == (2048, 1, 4, 4)


@pytest.mark.parametrize("which,depth,dhw", [("resnext3d", 101, (16, 112, 112)), ("resnext50_3d", 50, (32, 64, 64))])
def test_builtin_resnext3d_graph_equals_oracle(which, depth, dhw):
    """pooch_build_net(5 / 6) (host only) builds the oracle's task list: kinds, inputs, output
    shapes (C, D, H, W), kernel / stride / depth stride / padding and groups, task by task."""
    from paper_1907_05013_b200.executor import KINDS, build_net
    layers = build_net(which, dhw[1], 400, dhw[0])
    net = nets.resnext3d(dhw, classes=400, depth=depth)
    assert len(layers) == len(net.tasks)
    for d, t in zip(layers, net.tasks):
        assert KINDS[d.kind] == t.kind, t.name
        assert d.name.decode() == t.name
        assert [i for i in (d.in0, d.in1) if i >= 0] == [i for i in t.inputs if i >= 0], t.name
        shape = (d.cout, d.dout, d.hout, d.wout) if t.kind not in ("avgpool", "fc_ce") else (d.cout, 1, 1)
        assert shape == tuple(t.out_chw), t.name
        if t.kind in ("conv", "maxpool"):
            assert (d.k, d.stride, d.pad) == (t.k, t.stride, t.pad), t.name
            assert (d.stride_d or d.stride) == t.stride3[0], t.name
            assert max(d.groups, 1) == t.groups, t.name
