"""BN-ReLU prologue fusion on the GPU (POOCH_L_BNRELU_CONV).

The fused graph applies relu(BN(c)) to the consuming conv's operand on load with the BN-apply
kernel's arithmetic, so the conv sees bit-identical operands: one fused step must reproduce the
plain graph's step bit for bit (loss, every gradient, every updated parameter), match the fp64
oracle within 5e-3 (north_star), and every keep / swap / recompute plan of the fused graph must
be bit-exact against its in-core run.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthdata  # noqa: E402
from oracle import nets  # noqa: E402
from netutil import global_rel, load_params, pad_input, read_params  # noqa: E402

TOL = 5e-3
LR = 0.05


def _ctx(name, batch, in_hw, classes, dev_bytes, host_bytes, fuse):
    from paper_1907_05013_b200.executor import Context
    ctx = Context.builtin(name, batch, in_hw=in_hw, classes=classes, fuse=fuse)
    dev = torch.empty(dev_bytes, dtype=torch.uint8, device="cuda")
    host = torch.empty(host_bytes, dtype=torch.uint8, pin_memory=True)
    ctx.set_budget(dev, dev_bytes, host, host_bytes)
    ss = [torch.cuda.Stream() for _ in range(3)]
    ctx.set_streams(*ss)
    ctx._torch = (dev, host, ss)
    return ctx


def _step(ctx, params, x, t, strategy, fixed=None):
    load_params(ctx, params)
    dev = ctx._torch[0]
    xp, lp = ctx.input_slot()
    base = dev.data_ptr()
    xt = torch.from_numpy(pad_input(x)).reshape(-1).cuda()
    lt = torch.from_numpy(t.astype(np.int32)).cuda()
    dev[xp - base: xp - base + xt.numel() * 4].view(torch.float32).copy_(xt)
    dev[lp - base: lp - base + lt.numel() * 4].view(torch.int32).copy_(lt)
    torch.cuda.synchronize()
    cls, rep = ctx.plan(strategy, fixed=fixed)
    loss = ctx.train_step(LR)
    torch.cuda.synchronize()
    return loss, cls, rep


def _bits(ctx, which):
    return [ctx.get_param(i, which).view(np.uint32).copy() for i in range(len(ctx.params()))]


@pytest.fixture(scope="module", params=["tiny", "resnet50"])
def pair(request):
    if request.param == "tiny":
        net, b, hw, cls, dev, host = nets.tiny_cnn(), 8, 32, 10, 256 << 20, 64 << 20
        params = nets.init_params(net, seed=2, bn_random=True)
    else:
        net, b, hw, cls, dev, host = nets.resnet50(in_hw=224, classes=1000), 8, 224, 1000, 4 << 30, 2 << 30
        params = nets.init_params(net, seed=2, bn_random=True, residual_gamma=(0.1, 0.3))
    x = synthdata.images(b, hw, hw, 3, seed=0)
    t = synthdata.labels(b, cls, seed=1)
    plain = _ctx(request.param, b, hw, cls, dev, host, False)
    fused = _ctx(request.param, b, hw, cls, dev, host, True)
    plain.profile(1)
    fused.profile(1)
    return dict(name=request.param, net=net, params=params, x=x, t=t, plain=plain, fused=fused)


def test_fused_step_bit_identical_to_plain(pair):
    assert pair["fused"].n < pair["plain"].n                  # the conv-feeding BN-ReLU maps are gone
    l0, _, _ = _step(pair["plain"], pair["params"], pair["x"], pair["t"], "incore")
    g0, w0 = _bits(pair["plain"], 1), _bits(pair["plain"], 0)
    l1, _, _ = _step(pair["fused"], pair["params"], pair["x"], pair["t"], "incore")
    assert np.float32(l0).view(np.uint32) == np.float32(l1).view(np.uint32)
    for a, b, (name, _) in zip(_bits(pair["fused"], 1), g0, pair["fused"].params()):
        assert np.array_equal(a, b), name
    for a, b, (name, _) in zip(_bits(pair["fused"], 0), w0, pair["fused"].params()):
        assert np.array_equal(a, b), name


def test_fused_gradients_match_oracle(pair):
    ref_loss, ref_g, _ = nets.forward_backward(nets.fuse_bnrelu(pair["net"]), pair["params"], pair["x"], pair["t"])
    loss, _, _ = _step(pair["fused"], pair["params"], pair["x"], pair["t"], "incore")
    assert abs(loss - ref_loss) / abs(ref_loss) < TOL
    g = read_params(pair["fused"], pair["params"], 1)
    assert global_rel(g, ref_g) < TOL


def test_fused_plans_bit_exact(pair):
    ctx = pair["fused"]
    n = ctx.n
    ref_loss, _, _ = _step(ctx, pair["params"], pair["x"], pair["t"], "incore")
    ref_g = _bits(ctx, 1)
    g = synthdata.rng(9)
    f = [int(v) for v in g.integers(0, 3, n)]
    f[-1] = 1
    for strat, fixed in [("swap_all", None), ("fixed", [2] * (n - 1) + [1]), ("fixed", f)]:
        loss, cls, rep = _step(ctx, pair["params"], pair["x"], pair["t"], strat, fixed)
        assert np.float32(loss).view(np.uint32) == np.float32(ref_loss).view(np.uint32), strat
        for a, b in zip(_bits(ctx, 1), ref_g):
            assert np.array_equal(a, b), strat
