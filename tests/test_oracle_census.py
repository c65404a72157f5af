"""Pins for the saved-feature-map census (C2) against the paper's numbers."""
import json
import os

import numpy as np

from oracle import nets

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "census.json")))


def test_resnet50_has_105_maps_like_table3():
    net = nets.resnet50()
    assert len(nets.census(net, 1)) == GOLD["resnet50_maps"]
    for row in GOLD["table3_rows"]:
        assert sum(row) == GOLD["resnet50_maps"]


def test_resnet50_memory_claims():
    for v15 in (True, False):
        net = nets.resnet50(v15=v15)
        b640 = sum(b for _, b in nets.census(net, 640))
        assert b640 > GOLD["resnet50_batch640_min_bytes"]
        b256 = sum(b for _, b in nets.census(net, GOLD["incore_fails_from_batch"]))
        assert b256 > GOLD["v100_capacity_bytes"]


def test_resnet50_structure():
    net = nets.resnet50()
    kinds = [t.kind for t in net.tasks]
    assert kinds.count("conv") == 53
    assert kinds.count("bnrelu") + kinds.count("tail_id") + kinds.count("tail_proj") == 49
    assert sum(int(np.prod(s)) for s in nets.param_shapes(net).values()) == 25_557_032   # torchvision count
    assert net.tasks[-1].out_chw == (1000, 1, 1)
    assert net.tasks[-2].out_chw == (2048, 1, 1)


def test_tiny_cnn_census():
    net = nets.tiny_cnn()
    c = nets.census(net, 8)
    assert len(c) == 10
    assert sum(b for _, b in c) == 8 * 4 * (4 * 32 * 32 * 32 * 2 + 32 * 16 * 16 + 10)


def test_f2_fusion_census():
    """every bottleneck's two inner BN-ReLUs (and the tiny CNN's three
    conv-feeding ones) are applied on the consuming conv's operand load, so they stop being maps:
    ResNet-50 keeps 105 - 2 x 16 = 73 maps, the tiny CNN 10 - 3 = 7; the remaining maps are the
    plain graph's, bytes unchanged."""
    for net, dropped, n_f in ((nets.resnet50(), 32, 73), (nets.tiny_cnn(), 3, 7)):
        f = nets.fuse_bnrelu(net)
        assert len(f.tasks) == n_f == len(net.tasks) - dropped
        assert [t.kind for t in f.tasks].count("bnrelu_conv") == dropped
        plain = dict(nets.census(net, 640))
        fused = dict(nets.census(f, 640))
        gone = [t.name for t in net.tasks if t.kind == "bnrelu" and t.name not in fused]
        assert len(gone) == dropped
        assert all(fused[k] == plain[k] for k in fused)
        assert sum(plain.values()) - sum(fused.values()) == sum(plain[k] for k in gone)
        assert nets.param_shapes(f) == nets.param_shapes(net)       # same parameters, same order
    # the inner BN-ReLU outputs of ResNet-50 v1.5, per image, by hand (fp32, mid widths 64..512):
    # layer1 3 blocks x 2 x 56^2*64; layer2 56^2*128 (conv1 keeps 56^2 in v1.5) + 28^2*128 + 3 x 2 x
    # 28^2*128; layer3 28^2*256 + 14^2*256 + 5 x 2 x 14^2*256; layer4 14^2*512 + 7^2*512 + 2 x 2 x 7^2*512
    per_img = 4 * (6 * 56 * 56 * 64 + 56 * 56 * 128 + 7 * 28 * 28 * 128 + 28 * 28 * 256 + 11 * 14 * 14 * 256
                   + 14 * 14 * 512 + 5 * 7 * 7 * 512)
    assert per_img == 13_146_112
    r = nets.resnet50()
    gone = sum(b for (k, b), t in zip(nets.census(r, 640), r.tasks) if t.kind == "bnrelu" and k != "bn1")
    assert gone == 640 * per_img
    assert sum(b for _, b in nets.census(nets.fuse_bnrelu(r), 1)) == sum(b for _, b in nets.census(r, 1)) - per_img


def test_f2_fused_graph_computes_the_same_function():
    """The fused task is conv(relu(bn(c))) with the plain graph's operations in the same order, so
    loss and every gradient are identical in fp64 (tiny CNN and a 32x32 ResNet-50)."""
    import synthdata
    for net, hw, classes, b in ((nets.tiny_cnn(), 32, 10, 4), (nets.resnet50(in_hw=32, classes=10), 32, 10, 2)):
        params = nets.init_params(net, seed=2, bn_random=True)
        x = synthdata.images(b, hw, hw, 3, seed=0)
        t = synthdata.labels(b, classes, seed=1)
        l0, g0, _ = nets.forward_backward(net, params, x, t)
        l1, g1, _ = nets.forward_backward(nets.fuse_bnrelu(net), params, x, t)
        assert l0 == l1
        assert set(g0) == set(g1)
        for k in g0:
            assert np.array_equal(g0[k], g1[k]), k
