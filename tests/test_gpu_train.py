"""End-to-end GPU parity of the out-of-core training step (C ABI, cuda:0).

* gradients and loss of one step match the fp64 oracle within rel-L2 5e-3
  (BASELINE.json north_star) -- tiny CNN (config 1) and ResNet-50 at 224^2 --
  with the default 3xTF32 contractions (DESIGN.md Reading 27: with single
  TF32 operands the forward drifts ~1e-3 from fp64 and flips enough ReLU /
  max-pool decisions to move the gradients by O(1%); that mode is covered by
  the kernel-level tests and the bit-exactness test below);
* every keep / swap / recompute plan is bit-exact against the in-core run of
  the same kernels (north_star), including PoocH's plan at 50% of the in-core
  peak (config 1's budget) -- which also exercises the arena bound.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthdata  # noqa: E402
from oracle import nets  # noqa: E402
from netutil import global_rel, load_params, pad_input, read_params, rel  # noqa: E402

from gates import TOL, gate, gate_decided, gpu_decisions, step_for_decisions  # noqa: E402

LR = 0.05


def _ctx_for(name, batch, in_hw, classes, dev_bytes, host_bytes):
    from paper_1907_05013_b200.executor import Context
    ctx = Context.builtin(name, batch, in_hw=in_hw, classes=classes)
    dev = torch.empty(dev_bytes, dtype=torch.uint8, device="cuda")
    host = torch.empty(host_bytes, dtype=torch.uint8, pin_memory=True) if host_bytes else None
    ctx.set_budget(dev, dev_bytes, host, host_bytes)
    ss = [torch.cuda.Stream() for _ in range(3)]
    ctx.set_streams(*ss)
    ctx._torch = (dev, host, ss)
    return ctx


def _put_batch(ctx, x_nhwc, labels):
    dev = ctx._torch[0]
    xp, lp = ctx.input_slot()
    base = dev.data_ptr()
    xb = pad_input(x_nhwc)
    xt = torch.from_numpy(xb).reshape(-1).cuda()
    lt = torch.from_numpy(labels.astype(np.int32)).cuda()
    dev[xp - base: xp - base + xt.numel() * 4].view(torch.float32).copy_(xt)
    dev[lp - base: lp - base + lt.numel() * 4].view(torch.int32).copy_(lt)
    torch.cuda.synchronize()


def _step(ctx, params, x, t, strategy, fixed=None):
    load_params(ctx, params)
    _put_batch(ctx, x, t)
    cls, rep = ctx.plan(strategy, fixed=fixed)
    loss = ctx.train_step(LR)
    torch.cuda.synchronize()
    return loss, cls, rep


def _grads_bits(ctx):
    return [ctx.get_param(i, 1).view(np.uint32).copy() for i in range(len(ctx.params()))]


def _params_bits(ctx):
    return [ctx.get_param(i, 0).view(np.uint32).copy() for i in range(len(ctx.params()))]


@pytest.fixture(scope="module")
def tiny():
    net = nets.tiny_cnn()
    params = nets.init_params(net, seed=2, bn_random=True)
    x = synthdata.images(8, 32, 32, 3, seed=0)
    t = synthdata.labels(8, 10, seed=1)
    loss, grads, _ = nets.forward_backward(net, params, x, t)
    _, grads32, _ = nets.forward_backward(net, params, x, t, precision="fp32")
    ctx = _ctx_for("tiny", 8, 32, 10, 256 << 20, 64 << 20)
    ctx.profile(2)
    return dict(net=net, params=params, x=x, t=t, loss=loss, grads=grads, grads32=grads32, ctx=ctx)


def test_tiny_cnn_gradients_match_oracle(tiny):
    ctx = tiny["ctx"]
    loss, cls, rep = _step(ctx, tiny["params"], tiny["x"], tiny["t"], "incore")
    assert abs(loss - tiny["loss"]) / abs(tiny["loss"]) < TOL
    g = read_params(ctx, tiny["params"], 1)
    assert global_rel(g, tiny["grads"]) < TOL
    gate(g, tiny["grads"], tiny["grads32"], "tiny CNN")
    # the update: v = g, w' = w - lr * g on the first step (momentum starts at 0)
    w = read_params(ctx, tiny["params"], 0)
    ref_w, _ = nets.sgd_step(tiny["params"], {k: np.zeros_like(v) for k, v in tiny["params"].items()},
                             tiny["grads"], LR)
    assert global_rel(w, ref_w) < TOL


def test_tiny_cnn_plans_bit_exact(tiny):
    ctx = tiny["ctx"]
    n = ctx.n
    ref_loss, _, rep_in = _step(ctx, tiny["params"], tiny["x"], tiny["t"], "incore")
    ref_g, ref_w = _grads_bits(ctx), _params_bits(ctx)
    g = synthdata.rng(3)
    plans = [("swap_all", None), ("fixed", [2] * (n - 1) + [1]), ("fixed", [1] * n)]
    for _ in range(4):
        f = [int(v) for v in g.integers(0, 3, n)]
        f[-1] = min(f[-1], 1)
        plans.append(("fixed", f))
    for strat, fixed in plans:
        loss, cls, rep = _step(ctx, tiny["params"], tiny["x"], tiny["t"], strat, fixed)
        assert np.float32(loss).view(np.uint32) == np.float32(ref_loss).view(np.uint32), (strat, cls)
        for a, b in zip(_grads_bits(ctx), ref_g):
            assert np.array_equal(a, b), (strat, cls)
        for a, b in zip(_params_bits(ctx), ref_w):
            assert np.array_equal(a, b), (strat, cls)


def test_tiny_cnn_pooch_at_half_budget(tiny):
    """Config 1: budget = 50% of the in-core peak; PoocH must plan, stay in the
    arena and reproduce the in-core step bit for bit."""
    ctx = tiny["ctx"]
    ref, _, rep_in = _step(ctx, tiny["params"], tiny["x"], tiny["t"], "incore")
    ref_g = _grads_bits(ctx)
    peak = rep_in["peak_bytes"] + ctx.resident_bytes()
    half = ctx.resident_bytes() + rep_in["peak_bytes"] // 2
    half = (half + 255) // 256 * 256
    dev, host, ss = ctx._torch
    ctx.set_budget(dev, half, host, host.numel())
    ctx.profile(2)
    loss, cls, rep = _step(ctx, tiny["params"], tiny["x"], tiny["t"], "pooch")
    assert rep["feasible"] and rep["arena_bytes"] <= half
    assert cls != [0] * ctx.n                       # something had to leave the device
    assert np.float32(loss).view(np.uint32) == np.float32(ref).view(np.uint32)
    for a, b in zip(_grads_bits(ctx), ref_g):
        assert np.array_equal(a, b)
    ctx.set_budget(dev, dev.numel(), host, host.numel())
    ctx.profile(2)
    assert peak > half


def _r50_case(init):
    net = nets.resnet50(in_hw=224, classes=1000)
    if init == "small_residual":
        params = nets.init_params(net, seed=2, bn_random=True, residual_gamma=(0.1, 0.3))
    else:                                   # the bench's recipe: He-normal, gamma 1, beta 0
        params = nets.init_params(net, seed=2)
    x = synthdata.images(8, 224, 224, 3, seed=0)
    t = synthdata.labels(8, 1000, seed=1)
    loss, grads, _ = nets.forward_backward(net, params, x, t)
    _, grads32, _ = nets.forward_backward(net, params, x, t, precision="fp32")
    return dict(net=net, params=params, x=x, t=t, loss=loss, grads=grads, grads32=grads32)


@pytest.fixture(scope="module")
def r50():
    # 224^2 (the paper's input size) at batch 8; small-residual init (gamma3 ~ U(0.1, 0.3),
    # DESIGN.md Reading 28), where plain fp32 stays within 1.3e-3 of fp64 (whole gradient)
    d = _r50_case("small_residual")
    ctx = _ctx_for("resnet50", 8, 224, 1000, 4 << 30, 2 << 30)
    ctx.profile(1)
    d["ctx"] = ctx
    return d


def test_resnet50_gradients_match_oracle(r50):
    ctx = r50["ctx"]
    loss, cls, rep = _step(ctx, r50["params"], r50["x"], r50["t"], "incore")
    assert abs(loss - r50["loss"]) / abs(r50["loss"]) < TOL
    g = read_params(ctx, r50["params"], 1)
    assert global_rel(g, r50["grads"]) < TOL
    gate(g, r50["grads"], r50["grads32"], "ResNet-50 224^2 b8, small-residual init")


@pytest.mark.parametrize("which", ["tiny", "r50_small_residual", "r50_standard"])
def test_gradients_with_gpu_decisions(which, tiny, r50):
    """Reading 28: against the oracle taking the GPU's own ReLU masks and max-pool winners (read
    back from the step's maps), every gradient tensor is within the north_star's 5e-3 -- at the
    standard init too, where free-running fp32 itself is 2 % away."""
    if which == "tiny":
        d, ctx = tiny, tiny["ctx"]
    else:
        d = r50 if which == "r50_small_residual" else _r50_case("standard")
        ctx = r50["ctx"]
    step_for_decisions(ctx, lambda: _step(ctx, d["params"], d["x"], d["t"], "incore"))
    dec = gpu_decisions(ctx, d["net"])
    g = read_params(ctx, d["params"], 1)
    _, ref, _ = nets.forward_backward(d["net"], d["params"], d["x"], d["t"], decisions=dec)
    gate_decided(g, ref, which)


def test_resnet50_standard_init_gradients(r50):
    """The bench's own initialisation (gamma = 1, beta = 0): a chaotic random network in which
    plain fp32 alone moves the whole gradient 2.1 % from fp64 (the fp32 oracle; GPU: 3.9 %), so the
    whole-gradient gate is 3 x the fp32 oracle's and every tensor gets the fp32 floor (Reading 28);
    the loss still agrees to 5e-3."""
    d = _r50_case("standard")
    ctx = r50["ctx"]
    loss, cls, rep = _step(ctx, d["params"], d["x"], d["t"], "incore")
    assert abs(loss - d["loss"]) / abs(d["loss"]) < TOL
    g = read_params(ctx, d["params"], 1)
    assert global_rel(g, d["grads"]) <= max(TOL, 3.0 * global_rel(d["grads32"], d["grads"]))
    gate(g, d["grads"], d["grads32"], "ResNet-50 224^2 b8, standard init")


def test_resnet50_plans_bit_exact(r50):
    ctx = r50["ctx"]
    n = ctx.n
    ref_loss, _, _ = _step(ctx, r50["params"], r50["x"], r50["t"], "incore")
    ref_g = _grads_bits(ctx)
    g = synthdata.rng(5)
    f = [int(v) for v in g.integers(0, 3, n)]
    f[-1] = 1
    for strat, fixed in [("swap_all", None), ("fixed", [2] * (n - 1) + [0]), ("fixed", f)]:
        loss, cls, rep = _step(ctx, r50["params"], r50["x"], r50["t"], strat, fixed)
        assert np.float32(loss).view(np.uint32) == np.float32(ref_loss).view(np.uint32), strat
        for a, b in zip(_grads_bits(ctx), ref_g):
            assert np.array_equal(a, b), strat


def _nccl_uid():
    import ctypes
    lib = ctypes.CDLL("libnccl.so.2")
    raw = ctypes.create_string_buffer(128)
    assert lib.ncclGetUniqueId(raw) == 0
    return raw.raw


@pytest.mark.parametrize("net", ["tiny", "resnet50"])
def test_bucketed_allreduce_one_rank_is_identity(net):
    """the gradient allreduce runs in reverse-layer buckets on the comm stream,
    each gated by the backward that completes it, and SGD waits for the last one. With a 1-rank
    NCCL communicator the sum is the identity, so the step must be bit-identical to the run
    without a communicator -- this exercises the bucket boundaries, events and stream order
    on one GPU (the multi-rank sum is NCCL's)."""
    if net == "tiny":
        model = nets.tiny_cnn()
        batch, hw, classes, dev_b = 8, 32, 10, 256 << 20
        x, t = synthdata.images(8, 32, 32, 3, seed=0), synthdata.labels(8, 10, seed=1)
    else:
        model = nets.resnet50(in_hw=64, classes=100)
        batch, hw, classes, dev_b = 4, 64, 100, 2 << 30
        x, t = synthdata.images(4, 64, 64, 3, seed=0), synthdata.labels(4, 100, seed=1)
    params = nets.init_params(model, seed=2, bn_random=True)
    out = []
    for comm in (False, True):
        ctx = _ctx_for(net, batch, hw, classes, dev_b, 64 << 20)
        if comm:
            ctx.set_comm(_nccl_uid(), 0, 1)
        ctx.profile(1)
        loss, cls, _ = _step(ctx, params, x, t, "incore")
        out.append((np.float32(loss).view(np.uint32), _grads_bits(ctx), _params_bits(ctx)))
        ctx.close()
    assert out[0][0] == out[1][0]
    for a, b in zip(out[0][1] + out[0][2], out[1][1] + out[1][2]):
        assert np.array_equal(a, b)


def test_graph_replay_bit_identical_to_eager(tiny):
    """pooch_train_step replays the step as a captured CUDA graph; the instrumented (eager) step
    runs the same kernels in the same order, so loss, gradients and updated weights agree bit for
    bit -- for the step that captures the graph and for a later replay of it from the same state."""
    ctx = tiny["ctx"]
    _put_batch(ctx, tiny["x"], tiny["t"])
    ctx.plan("pooch")
    runs = []
    for timing in (True, False, False):             # eager, capture + launch, replay
        ctx.set_timing(timing)
        load_params(ctx, tiny["params"])
        loss = ctx.train_step(LR)
        torch.cuda.synchronize()
        runs.append((np.float32(loss).view(np.uint32), _grads_bits(ctx) + _params_bits(ctx)))
        assert ctx.step_was_graph() == (not timing)     # the replays really are graph launches
    ctx.set_timing(False)
    for loss, bits in runs[1:]:
        assert loss == runs[0][0]
        for a, b in zip(bits, runs[0][1]):
            assert np.array_equal(a, b)


def test_profiling_modes(tiny):
    """Sec. 4.2: with a host arena that holds every map, pooch_profile measures real all-swap
    iterations (per-task times under the copy traffic, every swapped map's copy time and issue time);
    with an undersized host arena AUTO falls back to isolated timing and ALL_SWAP refuses."""
    from paper_1907_05013_b200._lib import PoochError
    ctx = tiny["ctx"]
    dev, host, ss = ctx._torch
    _put_batch(ctx, tiny["x"], tiny["t"])
    ctx.set_profile_mode("auto")
    p = ctx.profile(2)
    assert p["mode"] == "all_swap" and p["step_ns"] > 0
    swapped = [m for m in range(ctx.n) if p["d2h_issue"][m] >= 0]
    assert swapped and all(p["h2d_issue"][m] > p["d2h_issue"][m] for m in swapped)
    assert all(v > 0 for v in p["fwd"] + p["bwd"])
    cls, rep = ctx.plan("pooch")                 # plans from the all-swap profile
    assert rep["feasible"]
    small = 4096
    ctx.set_budget(dev, dev.numel(), host, small)   # host arena far below the maps
    load_params(ctx, tiny["params"])
    _put_batch(ctx, tiny["x"], tiny["t"])
    assert ctx.profile(1)["mode"] == "isolated"
    ctx.set_profile_mode("all_swap")
    with pytest.raises(PoochError) as e:
        ctx.profile(1)
    assert e.value.status == 2
    ctx.set_profile_mode("auto")
    ctx.set_budget(dev, dev.numel(), host, host.numel())
    load_params(ctx, tiny["params"])
    ctx.profile(2)


def test_measured_trace_and_plan_from_a_faster_link(tiny):
    """(1) pooch_last_trace: the executed timeline of an instrumented step -- compute ops in
    program order without overlap, each swap-in after its swap-out. (2) The paper's portability
    experiment (a plan made for the faster POWER9 link ran out of memory on x86): a plan
    made from a profile claiming an 8x faster host link, executed on the real one, cannot overrun
    the arena (static offsets + event-ordered reuse) and reproduces the in-core step bit for bit;
    it is only slower than its simulation promised."""
    ctx = tiny["ctx"]
    ref, _, rep_in = _step(ctx, tiny["params"], tiny["x"], tiny["t"], "incore")
    ref_g = _grads_bits(ctx)
    dev, host, ss = ctx._torch
    half = (ctx.resident_bytes() + rep_in["peak_bytes"] // 2 + 255) // 256 * 256
    ctx.set_budget(dev, half, host, host.numel())
    load_params(ctx, tiny["params"])
    _put_batch(ctx, tiny["x"], tiny["t"])
    ctx.set_profile_mode("isolated")
    p = ctx.profile(2)
    fast = [max(1, v // 8) for v in p["d2h"]], [max(1, v // 8) for v in p["h2d"]]
    ctx.set_profile(p["fwd"], p["bwd"], p["rec"], fast[0], fast[1], p["tail"])
    load_params(ctx, tiny["params"])
    cls, rep = ctx.plan("swap_all")
    assert rep["arena_bytes"] <= half
    ctx.set_timing(True)
    loss = ctx.train_step(LR)
    torch.cuda.synchronize()
    tr = ctx.last_trace()
    ctx.set_timing(False)
    assert np.float32(loss).view(np.uint32) == np.float32(ref).view(np.uint32)
    for a, b in zip(_grads_bits(ctx), ref_g):
        assert np.array_equal(a, b)
    comp = [e for e in tr if e[0] == "COMPUTE"]
    assert all(a[4] <= b[3] + 1000 for a, b in zip(comp, comp[1:]))   # serial on the compute lane
    outs = {e[2]: e for e in tr if e[1] == "O"}
    ins = {e[2]: e for e in tr if e[1] == "I"}
    assert ins and all(ins[m][3] >= outs[m][4] - 1000 for m in ins)   # swap-in after its swap-out
    ctx.set_profile_mode("auto")
    ctx.set_budget(dev, dev.numel(), host, host.numel())
    load_params(ctx, tiny["params"])
    ctx.profile(2)


def test_poisoned_frees_stay_bit_exact(tiny):
    """SURVEY 5 debug mode: with POOCH_DEBUG_POISON=1 every freed buffer instance is NaN-filled on
    its stream right after the freeing op, so any read after a free (a missing cross-stream wait,
    an overlapping offset) would poison the step. Every plan of the bit-exactness test, including
    PoocH at half the in-core peak, still reproduces the unpoisoned in-core step bit for bit."""
    import os
    ctx = tiny["ctx"]
    n = ctx.n
    ref_loss, _, rep_in = _step(ctx, tiny["params"], tiny["x"], tiny["t"], "incore")
    ref_g = _grads_bits(ctx)
    g = synthdata.rng(13)
    plans = [("swap_all", None), ("fixed", [2] * (n - 1) + [1])]
    for _ in range(3):
        f = [int(v) for v in g.integers(0, 3, n)]
        f[-1] = min(f[-1], 1)
        plans.append(("fixed", f))
    os.environ["POOCH_DEBUG_POISON"] = "1"
    try:
        for strat, fixed in plans:
            loss, cls, rep = _step(ctx, tiny["params"], tiny["x"], tiny["t"], strat, fixed)
            assert np.float32(loss).view(np.uint32) == np.float32(ref_loss).view(np.uint32), (strat, cls)
            for a, b in zip(_grads_bits(ctx), ref_g):
                assert np.array_equal(a, b), (strat, cls)
        dev, host, ss = ctx._torch
        half = (ctx.resident_bytes() + rep_in["peak_bytes"] // 2 + 255) // 256 * 256
        ctx.set_budget(dev, half, host, host.numel())
        load_params(ctx, tiny["params"])
        _put_batch(ctx, tiny["x"], tiny["t"])
        ctx.profile(2)
        loss, cls, rep = _step(ctx, tiny["params"], tiny["x"], tiny["t"], "pooch")
        assert np.float32(loss).view(np.uint32) == np.float32(ref_loss).view(np.uint32)
        for a, b in zip(_grads_bits(ctx), ref_g):
            assert np.array_equal(a, b)
    finally:
        os.environ.pop("POOCH_DEBUG_POISON", None)
    ctx.set_budget(dev, dev.numel(), host, host.numel())
    load_params(ctx, tiny["params"])
    ctx.profile(2)
