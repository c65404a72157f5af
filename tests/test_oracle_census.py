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
