"""GPU parity of the AlexNet workload against the fp64 oracle.

* LRN forward / backward through pooch_op_lrn_* (C = 96 and 256, ragged pixel counts);
* one training step of AlexNet (in-core plan) against oracle/nets.py at 67x67 and at the paper's
  227x227 input: loss, and every gradient under Reading 28's gate; the dropout masks (counter-based,
  pooch_set_rng) equal the oracle's exactly, and the step counter advances per step;
* keep / swap / recompute plans are bit-exact against the in-core step (north_star), including
  PoocH's plan at 70 % of the in-core peak."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthdata  # noqa: E402
from gates import TOL, gate, gate_decided, gpu_decisions, step_for_decisions  # noqa: E402
from netutil import global_rel, load_params, pad_input, read_params, rel  # noqa: E402
from oracle import layers as L  # noqa: E402
from oracle import nets  # noqa: E402

LR = 0.01
SEED, STEP = 5, 3


def _lib():
    from paper_1907_05013_b200 import _lib
    return _lib


def ptr(t):
    return C.c_void_p(t.data_ptr())


@pytest.mark.parametrize("pixels,ch", [(37, 96), (129, 256), (16, 256)])
def test_lrn_op(pixels, ch):
    lib = _lib()
    g = synthdata.rng(pixels + ch)
    x = (g.standard_normal((pixels, ch)) * 40.0).astype(np.float32)
    gy = g.standard_normal((pixels, ch)).astype(np.float32)
    dx, dgy = torch.from_numpy(x).cuda(), torch.from_numpy(gy).cuda()
    y, gx = torch.empty_like(dx), torch.empty_like(dx)
    lib.check(lib.lib.pooch_op_lrn_fwd(ptr(dx), ptr(y), pixels, ch, None))
    lib.check(lib.lib.pooch_op_lrn_bwd(ptr(dx), ptr(dgy), ptr(gx), pixels, ch, None))
    torch.cuda.synchronize()
    x4 = x.T[None, :, :, None].astype(np.float64)            # NCHW with H = pixels, W = 1
    ref_y = L.lrn_fwd(x4)[0][0, :, :, 0].T
    ref_gx = L.lrn_bwd(gy.T[None, :, :, None].astype(np.float64), x4)[0, :, :, 0].T
    assert rel(y.cpu().numpy(), ref_y) < 1e-6
    assert rel(gx.cpu().numpy(), ref_gx) < 1e-6


def _ctx(batch, hw, dev_bytes, host_bytes):
    from paper_1907_05013_b200.executor import Context
    ctx = Context.builtin("alexnet", batch, in_hw=hw)
    dev = torch.empty(dev_bytes, dtype=torch.uint8, device="cuda")
    host = torch.empty(host_bytes, dtype=torch.uint8, pin_memory=True)
    ctx.set_budget(dev, dev_bytes, host, host_bytes)
    ss = [torch.cuda.Stream() for _ in range(3)]
    ctx.set_streams(*ss)
    ctx._torch = (dev, host, ss)
    return ctx


def _put(ctx, x, t):
    dev = ctx._torch[0]
    xp, lp = ctx.input_slot()
    base = dev.data_ptr()
    xt = torch.from_numpy(pad_input(x)).reshape(-1).cuda()
    lt = torch.from_numpy(t.astype(np.int32)).cuda()
    dev[xp - base: xp - base + xt.numel() * 4].view(torch.float32).copy_(xt)
    dev[lp - base: lp - base + lt.numel() * 4].view(torch.int32).copy_(lt)
    torch.cuda.synchronize()


def _case(hw, batch):
    net = nets.alexnet(in_hw=hw)
    params = nets.init_params(net, seed=2)
    g = synthdata.rng(4)
    for k in params:
        if k.endswith(".b"):
            params[k] = g.uniform(-0.05, 0.05, params[k].shape).astype(np.float32)
    x = synthdata.images(batch, hw, hw, 3, seed=0)
    t = synthdata.labels(batch, 1000, seed=1)
    loss, grads, outs = nets.forward_backward(net, params, x, t, rng=(SEED, STEP))
    _, grads32, _ = nets.forward_backward(net, params, x, t, precision="fp32", rng=(SEED, STEP))
    return dict(net=net, params=params, x=x, t=t, loss=loss, grads=grads, grads32=grads32, outs=outs)


def _step(ctx, d, strategy, fixed=None):
    load_params(ctx, d["params"])
    _put(ctx, d["x"], d["t"])
    ctx.set_rng(SEED, STEP)
    cls, rep = ctx.plan(strategy, fixed=fixed)
    loss = ctx.train_step(LR)
    torch.cuda.synchronize()
    return loss, cls, rep


@pytest.fixture(scope="module")
def small():
    d = _case(67, 4)
    d["ctx"] = _ctx(4, 67, 1536 << 20, 64 << 20)
    d["ctx"].profile(1)
    return d


def test_alexnet_step_matches_oracle(small):
    ctx = small["ctx"]
    loss, cls, rep = _step(ctx, small, "incore")
    assert abs(loss - small["loss"]) / abs(small["loss"]) < TOL
    g = read_params(ctx, small["params"], 1)
    assert global_rel(g, small["grads"]) < TOL
    gate(g, small["grads"], small["grads32"], "AlexNet 67^2 b4")
    step_for_decisions(ctx, lambda: _step(ctx, small, "incore"))
    dec = gpu_decisions(ctx, small["net"])
    _, ref, _ = nets.forward_backward(small["net"], small["params"], small["x"], small["t"], rng=(SEED, STEP),
                                      decisions=dec)
    gate_decided(read_params(ctx, small["params"], 1), ref, "AlexNet 67^2 b4")


def test_dropout_masks_equal_the_oracle_and_advance(small):
    """The GPU draws the oracle's masks: fc7's weight gradient dW7 = dz7^T y6 has an all-zero column
    exactly where fc6's output is zero in every row (dropped or non-positive); and the step counter
    advances -- a second step from the same weights, without pooch_set_rng, matches the oracle at
    step + 1 (a different mask), not at step."""
    ctx = small["ctx"]
    net = small["net"]
    _step(ctx, small, "incore")
    fc6 = [i for i, t in enumerate(net.tasks) if t.name == "fc6"][0]
    y6 = small["outs"][fc6][:, :, 0, 0]
    g = read_params(ctx, small["params"], 1)
    dead = np.all(y6 == 0, axis=0)
    assert dead.any() and (~dead).any()
    assert np.all(g["fc7.w"][:, dead] == 0)
    assert np.all(np.any(g["fc7.w"][:, ~dead] != 0, axis=0))
    load_params(ctx, small["params"])                # same weights, counter now STEP + 1
    ctx.train_step(LR)
    torch.cuda.synchronize()
    g2 = read_params(ctx, small["params"], 1)
    loss2, ref2, _ = nets.forward_backward(net, small["params"], small["x"], small["t"], rng=(SEED, STEP + 1))
    assert global_rel(g2, ref2) < TOL
    assert global_rel(g2, small["grads"]) > 10 * TOL


def test_alexnet_plans_bit_exact(small):
    ctx = small["ctx"]
    n = ctx.n
    ref_loss, _, rep_in = _step(ctx, small, "incore")
    ref_g = [ctx.get_param(i, 1).view(np.uint32).copy() for i in range(len(ctx.params()))]
    g = synthdata.rng(9)
    f = [int(v) for v in g.integers(0, 3, n)]
    f[-1] = 1
    for strat, fixed in [("swap_all", None), ("fixed", [2] * (n - 1) + [0]), ("fixed", f)]:
        loss, cls, rep = _step(ctx, small, strat, fixed)
        assert np.float32(loss).view(np.uint32) == np.float32(ref_loss).view(np.uint32), strat
        for a, b in zip([ctx.get_param(i, 1).view(np.uint32) for i in range(len(ctx.params()))], ref_g):
            assert np.array_equal(a, b), strat
    # PoocH below the in-core peak: the widest task (LRN1: conv1's map, its output and both
    # gradients) needs 4 x the largest map, most of AlexNet's peak at this size
    dev, host, ss = ctx._torch
    widest = int(4 * max(4 * np.prod(t.out_chw) * 4 for t in small["net"].tasks))
    half = (ctx.resident_bytes() + (widest + rep_in["peak_bytes"]) // 2 + 255) // 256 * 256
    assert half < ctx.resident_bytes() + rep_in["peak_bytes"]
    ctx.set_budget(dev, half, host, host.numel())
    load_params(ctx, small["params"])
    _put(ctx, small["x"], small["t"])
    ctx.profile(1)
    loss, cls, rep = _step(ctx, small, "pooch")
    assert rep["feasible"] and rep["arena_bytes"] <= half and cls != [0] * n
    assert np.float32(loss).view(np.uint32) == np.float32(ref_loss).view(np.uint32)
    for a, b in zip([ctx.get_param(i, 1).view(np.uint32) for i in range(len(ctx.params()))], ref_g):
        assert np.array_equal(a, b)
    ctx.set_budget(dev, dev.numel(), host, host.numel())


def test_alexnet_227_step_matches_oracle():
    """The paper's 227 x 227 input, batch 2. Free-running, the whole gradient is within 5e-3, but
    conv1 / conv2 carry max-pool winner flips over the 2 x 256 x 27 x 27 overlapping windows (an
    fp64 oracle with 2e-5 relative noise on its contraction outputs moves conv1.w by 2.8e-2,
    tools/noise_conditioning.py); with the GPU's own decisions every tensor is within 5e-3."""
    d = _case(227, 2)
    ctx = _ctx(2, 227, 3 << 30, 64 << 20)
    ctx.profile(1)
    loss, cls, rep = step_for_decisions(ctx, lambda: _step(ctx, d, "incore"))
    assert abs(loss - d["loss"]) / abs(d["loss"]) < TOL
    g = read_params(ctx, d["params"], 1)
    assert global_rel(g, d["grads"]) < TOL
    dec = gpu_decisions(ctx, d["net"])
    _, ref, _ = nets.forward_backward(d["net"], d["params"], d["x"], d["t"], rng=(SEED, STEP), decisions=dec)
    gate_decided(g, ref, "AlexNet 227^2 b2")
    ctx.close()
