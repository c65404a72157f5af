"""The C-ABI library loads on a CPU-only box and exports every symbol that
include/pooch.h declares; host-only entry points validate their arguments."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "pooch.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pooch_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    from paper_1907_05013_b200 import _lib
    names = declared()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(_lib.lib, n)]
    assert not missing, missing
    unbound = [n for n in names if n not in _lib.SIGNATURES]
    assert not unbound, unbound


def test_build_net_census_matches_oracle():
    from oracle import nets
    from paper_1907_05013_b200.executor import build_net, KINDS
    for which, ref in (("resnet50", nets.resnet50()), ("tiny", nets.tiny_cnn())):
        layers = build_net(which, 224 if which == "resnet50" else 32, 1000 if which == "resnet50" else 10)
        assert len(layers) == len(ref.tasks)
        for l, t in zip(layers, ref.tasks):
            assert l.name.decode() == t.name
            assert KINDS[l.kind] == t.kind
            assert [i for i in (l.in0, l.in1) if i >= 0] == [i for i in t.inputs if i >= 0]
            assert (l.cout, l.hout, l.wout) == t.out_chw
            if t.kind == "conv":
                assert (l.k, l.stride, l.pad) == (t.k, t.stride, t.pad)


def test_create_validates_graph_without_gpu():
    from paper_1907_05013_b200 import _lib
    from paper_1907_05013_b200.executor import Context, build_net
    layers = build_net("tiny", 32, 10)
    layers[3].in0 = 5                               # not topological
    with pytest.raises(_lib.PoochError) as e:
        Context(layers, 8, 4, 32, 32, 10)
    assert e.value.status == 1
    ctx = Context(build_net("tiny", 32, 10), 8, 4, 32, 32, 10)     # host-only: no device work
    names = [n for n, _ in ctx.params()]
    assert names[0] == "conv0.w" and names[-1] == "fc.b"
    assert dict(ctx.params())["fc.w"] == 12 * 8192                 # classes padded 10 -> 12
    assert ctx.resident_bytes() > 0
    ctx.close()


def test_plan_problem_errors():
    from paper_1907_05013_b200.planning import PlanProblem
    p = PlanProblem([1] * 13, [1] * 13, [4] * 13, [1] * 13, [1] * 13, [[]] + [[i] for i in range(12)],
                    [[i] for i in range(13)])
    from paper_1907_05013_b200 import _lib
    with pytest.raises(_lib.PoochError):
        p.plan("exhaustive")                        # n > 12 is a usage error
    p2 = PlanProblem([1, 1], [1, 1], [4, 4], [1, 1], [1, 1], [[], [0]], [[0], [0, 1]], resident=10, budget=12)
    cls, rep = p2.plan("pooch")
    assert cls is None and rep.feasible == 0        # nothing fits: EINFEASIBLE


def test_unet3d_graph_matches_oracle_without_gpu():
    """Config 4's 3D U-Net: the C builder's tasks equal the oracle's (names, kinds, inputs,
    shapes), and a context for it is created host-only with every map of the oracle's size."""
    from oracle import nets
    from paper_1907_05013_b200.executor import KINDS, Context, build_net
    ref = nets.unet3d(in_d=32, width=32, classes=2)
    layers = build_net("unet3d", 32, 2, 32)
    assert len(layers) == len(ref.tasks) == 45
    for l, t in zip(layers, ref.tasks):
        assert l.name.decode() == t.name
        assert KINDS[l.kind] == t.kind
        assert [i for i in (l.in0, l.in1) if i >= 0] == [i for i in t.inputs if i >= 0]
        assert (l.cout, l.dout, l.hout, l.wout) == t.out_chw
    ctx = Context.builtin("unet3d", 1, in_hw=32, classes=2, width=32)
    prob = ctx.plan_problem() if hasattr(ctx, "plan_problem") else None
    names = dict(ctx.params())
    assert names["up1.w"] == 64 * 8 * 32 and names["enc1.conv1.w"] == 32 * 27 * 32   # Cin padded 1 -> 32
    assert names["head.w"] == 4 * 32                                                   # classes padded 2 -> 4
    ctx.close()
    bad = build_net("unet3d", 32, 2, 32)
    with pytest.raises(Exception):
        Context(bad, 2, 32, 32, 32, 2, in_d=32)          # 3D networks run at batch 1


def test_allreduce_buckets_partition_the_gradient_region():
    """The per-bucket allreduce ranges tile the gradient region exactly (no gap, no overlap),
    in reverse-layer order, each closed by the lowest-index task whose parameters it holds."""
    from paper_1907_05013_b200.executor import Context, build_net
    ctx = Context(build_net("resnet50", 224, 1000), 8, 4, 224, 224, 1000)
    total = sum((numel + 3) // 4 * 4 for _, numel in ctx.params())
    b = ctx.allreduce_buckets()
    assert len(b) >= 3
    assert b[0][1] == total and b[-1][0] == 0                 # first bucket = the network's tail
    for (lo1, hi1, t1), (lo2, hi2, t2) in zip(b, b[1:]):
        assert hi2 == lo1 and t2 < t1                         # contiguous, descending
    assert all(hi - lo >= 6_500_000 for lo, hi, _ in b[:-1])
    ctx.close()


def test_fused_build_net_matches_oracle_and_keeps_parameters():
    """the C++ builder's BN-ReLU fusion (POOCH_NET_FUSE_BNRELU) produces the
    oracle's fused graph (nets.fuse_bnrelu) task for task, and the fused context has exactly the
    plain context's parameters in the same order (host-only, no device work)."""
    from oracle import nets
    from paper_1907_05013_b200.executor import KINDS, Context, build_net
    for which, ref, hw, cls in (("resnet50", nets.resnet50(), 224, 1000), ("tiny", nets.tiny_cnn(), 32, 10)):
        f = nets.fuse_bnrelu(ref)
        layers = build_net(which, hw, cls, fuse=True)
        assert len(layers) == len(f.tasks)
        for l, t in zip(layers, f.tasks):
            assert KINDS[l.kind] == t.kind
            assert l.name.decode() == (t.bn + "+" + t.name if t.kind == "bnrelu_conv" else t.name)
            assert [i for i in (l.in0, l.in1) if i >= 0] == [i for i in t.inputs if i >= 0]
            assert (l.cout, l.hout, l.wout) == t.out_chw
        a = Context(build_net(which, hw, cls), 2, 4, hw, hw, cls)
        b = Context(layers, 2, 4, hw, hw, cls)
        assert a.params() == b.params()
        assert sum(n for _, n in a.params()) == sum(n for _, n in b.params())
        a.close()
        b.close()
