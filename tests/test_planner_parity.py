"""The C++ simulator and planner (libpooch.so, host-only calls) against the
oracle: identical timelines (tolerance 0) and identical class vectors."""
import json
import os

import numpy as np
import pytest

import synthdata
from oracle import nets, planner as OP, sim as OS

pp = pytest.importorskip("paper_1907_05013_b200.planning")

G = os.path.join(os.path.dirname(__file__), "golden")


def both(d, **kw):
    return OS.Profile.from_dict(d, **kw), pp.PlanProblem.from_dict(d, **kw)


def _cmp_sim(po, pc, cls, sched):
    ro = OS.simulate(po, cls, sched)
    rc = pc.simulate(cls, sched, events=True)
    assert rc["oom"] == ro.oom
    assert rc["peak"] == ro.peak or ro.oom
    if ro.oom:
        return ro
    assert rc["makespan"] == ro.makespan
    assert rc["events"] == [tuple(e) for e in ro.events]
    assert rc["L_O"] == ro.L_O and rc["L_I"] == ro.L_I
    assert rc["stall"] == ro.stall
    return ro


def test_spec_and_fig11_through_cabi():
    d = json.load(open(os.path.join(G, "spec_traces.json")))
    _, pc = both(d["profile"])
    assert pc.simulate([OS.KEEP])["makespan"] == d["keep_makespan"]
    assert pc.simulate([OS.SWAP])["makespan"] == d["swap_makespan"]
    f = json.load(open(os.path.join(G, "fig11_chain.json")))
    _, pc = both(f)
    r = pc.simulate([OS.SWAP] * 8)
    assert sorted(r["L_O"]) == f["L_O"] and sorted(r["L_I"]) == f["L_I"]


@pytest.mark.parametrize("seed", range(60))
def test_sim_differential(seed):
    g = synthdata.rng(500 + seed)
    n = int(g.integers(1, 9))
    d = synthdata.random_profile(n, seed, dag=seed % 2 == 0)
    budget = int(10 + sum(d["bytes"]) * g.uniform(0.3, 1.6))
    po, pc = both(d, resident=10, budget=budget)
    for _ in range(8):
        cls = [int(c) for c in g.integers(0, 4, n)]
        if cls[-1] == OS.RECOMPUTE:
            cls[-1] = OS.SWAP
        for sched in (OS.EAGER, OS.NAIVE):
            _cmp_sim(po, pc, cls, sched)


@pytest.mark.parametrize("seed", range(40))
def test_sim_differential_shared_link(seed):
    """Reading 51: copies slowed while both copy lanes are busy -- same timelines, tolerance 0."""
    g = synthdata.rng(700 + seed)
    n = int(g.integers(1, 9))
    d = synthdata.random_profile(n, seed, dag=seed % 2 == 1)
    budget = int(10 + sum(d["bytes"]) * g.uniform(0.5, 1.8))
    dx = (int(g.integers(300, 1001)), int(g.integers(300, 1001)))
    po, pc = both(d, resident=10, budget=budget, duplex=dx)
    for _ in range(8):
        cls = [int(c) for c in g.integers(0, 4, n)]
        if cls[-1] == OS.RECOMPUTE:
            cls[-1] = OS.SWAP
        for sched in (OS.EAGER, OS.NAIVE, OS.SN):
            _cmp_sim(po, pc, cls, sched)


@pytest.mark.parametrize("seed", range(12))
def test_pooch_identical_to_oracle_shared_link(seed):
    d, budget = _tight(seed + 100, 6 + seed % 5)
    dx = (750 + 10 * seed, 760)
    po, pc = both(d, resident=10, budget=budget, duplex=dx)
    ref = OP.pooch(po, li_cap=16)
    cls, rep = pc.plan("pooch", threads=4)
    if not ref["feasible"]:
        assert cls is None
        return
    assert cls == ref["cls"]
    assert rep.makespan_ns == ref["makespan"]


def _tight(seed, n):
    d = synthdata.random_profile(n, seed, dag=seed % 3 == 0)
    g = synthdata.rng(91 + seed)
    budget = 10 + max(3 * max(d["bytes"]), int(sum(d["bytes"]) * g.uniform(0.45, 0.95)))
    return d, budget


@pytest.mark.parametrize("seed", range(30))
def test_pooch_identical_to_oracle(seed):
    d, budget = _tight(seed, 6 + seed % 7)
    po, pc = both(d, resident=10, budget=budget)
    ref = OP.pooch(po, li_cap=16)
    cls, rep = pc.plan("pooch", threads=4)
    if not ref["feasible"]:
        assert cls is None
        return
    assert cls == ref["cls"]
    assert rep.makespan_ns == ref["makespan"]


@pytest.mark.parametrize("seed", range(8))
def test_exhaustive_equals_brute_force(seed):
    d, budget = _tight(seed, 5 + seed % 3)
    po, pc = both(d, resident=10, budget=budget)
    bf = OP.brute_force(po)
    cls, rep = pc.plan("exhaustive", threads=4)
    assert cls == bf["cls"]
    if cls is not None:
        assert rep.makespan_ns == bf["makespan"]


def _net_profile(net, batch, link_gbs, budget, scale_ns=1.0):
    """Synthetic per-task times for a real graph: compute ~ flops, copies ~ bytes / link."""
    n = len(net.tasks)
    fwd, nbytes = [], []
    for i, t in enumerate(net.tasks):
        b = batch * net.map_bytes_per_image(i)
        nbytes.append(b)
        if t.kind in ("conv", "bnrelu_conv"):
            c, h, w = t.out_chw
            fl = 2 * batch * c * h * w * t.cin * t.k * t.k
            fwd.append(max(1, int(fl / 300e3 * scale_ns)))      # ~300 TFLOP/s
        else:
            fwd.append(max(1, int(3 * b / 6e3 * scale_ns)))     # ~6 TB/s, 3 passes
    bwd = [2 * f for f in fwd]
    x = [max(1, int(b / link_gbs)) for b in nbytes]
    inputs = [[j for j in t.inputs if j >= 0] for t in net.tasks]
    needs = [net.needs(i) for i in range(n)]
    d = dict(fwd=fwd, bwd=bwd, bytes=nbytes, d2h=x, h2d=x, inputs=inputs, needs=needs)
    return d


@pytest.mark.parametrize("link", [16.0, 75.0])
def test_tiny_cnn_profile_parity(link):
    net = nets.tiny_cnn()
    d = _net_profile(net, 8, link, 0)
    total = sum(d["bytes"])
    po, pc = both(d, resident=1_500_000, budget=1_500_000 + total // 2)
    ref = OP.pooch(po, li_cap=16)
    cls, _ = pc.plan("pooch")
    assert cls == (ref["cls"] if ref["feasible"] else None)
    bf = OP.brute_force(po)
    if bf["cls"] is not None and ref["feasible"]:
        assert ref["makespan"] >= bf["makespan"]


@pytest.mark.parametrize("link", [16.0, 75.0])
def test_resnet50_profile_parity_small_cap(link):
    """Full 105-task ResNet-50 graph at batch 64; li_cap 3 keeps the oracle fast."""
    net = nets.resnet50()
    d = _net_profile(net, 64, link, 0)
    total = sum(d["bytes"])
    po, pc = both(d, resident=200_000_000, budget=200_000_000 + int(total * 0.35))
    for cls in ([OS.SWAP] * 105, [OS.KEEP] * 105):
        _cmp_sim(po, pc, cls, OS.EAGER)
    ref = OP.pooch(po, li_cap=3)
    cls, rep = pc.plan("pooch", li_cap=3)
    assert cls == (ref["cls"] if ref["feasible"] else None)


@pytest.mark.parametrize("seed", range(25))
def test_superneurons_sched_differential(seed):
    g = synthdata.rng(900 + seed)
    n = int(g.integers(2, 9))
    d = synthdata.random_profile(n, seed, dag=seed % 2 == 0)
    d["is_conv"] = [int(v) for v in g.integers(0, 2, n)]
    budget = int(10 + sum(d["bytes"]) * g.uniform(0.3, 1.6))
    po, pc = both(d, resident=10, budget=budget)
    for _ in range(6):
        cls = [int(c) for c in g.integers(0, 3, n)]
        cls[-1] = min(cls[-1], OS.SWAP)
        _cmp_sim(po, pc, cls, OS.SN)
    ref_cls, ref_ms = OP.superneurons(po)
    cls, rep = pc.plan("superneurons")
    if ref_ms == OP.INF:
        assert cls is None
    else:
        assert cls == ref_cls and rep.makespan_ns == ref_ms


def test_superneurons_rule_on_resnet50_census():
    """Table 3's SuperNeurons row has the same counts on both machines:
    the rule depends only on sizes and layer types, never on the link."""
    net = nets.resnet50()
    counts = []
    for link in (16.0, 75.0):
        d = _net_profile(net, 512, link, 0)
        d["is_conv"] = [int(t.kind == "conv") for t in net.tasks]
        po = OS.Profile.from_dict(d, resident=2_000_000_000, budget=16_000_000_000)
        cls, _ = OP.superneurons(po)
        counts.append((cls.count(OS.KEEP), cls.count(OS.SWAP), cls.count(OS.RECOMPUTE)))
    assert counts[0] == counts[1]
    assert sum(counts[0]) == 105


@pytest.mark.parametrize("seed", range(10))
def test_host_budget_limits_swap_class(seed):
    d, budget = _tight(seed, 8)
    hb = sum(d["bytes"]) // 3
    po, pc = both(d, resident=10, budget=budget, host_budget=hb)
    ref = OP.pooch(po, li_cap=16)
    cls, rep = pc.plan("pooch")
    if not ref["feasible"]:
        assert cls is None
        return
    assert cls == ref["cls"]
    assert sum(d["bytes"][m] for m in range(8) if cls[m] == OS.SWAP) <= hb
    assert pc.simulate([OS.SWAP] * 8)["oom"]          # all-swap needs more host memory than hb


@pytest.mark.parametrize("link", [16.0, 75.0])
def test_fused_graphs_profile_parity(link):
    """the C++ planner matches the oracle on the BN-ReLU-fused graphs too (tiny CNN:
    7 maps, full tree; ResNet-50: 73 maps, li_cap 3), and the tiny graph's PoocH plan is no better
    than brute force over all 2 * 3^6 plans."""
    tiny = nets.fuse_bnrelu(nets.tiny_cnn())
    d = _net_profile(tiny, 8, link, 0)
    total = sum(d["bytes"])
    po, pc = both(d, resident=1_500_000, budget=1_500_000 + total // 2)
    ref = OP.pooch(po, li_cap=16)
    cls, _ = pc.plan("pooch")
    assert cls == (ref["cls"] if ref["feasible"] else None)
    bf = OP.brute_force(po)
    if bf["cls"] is not None and ref["feasible"]:
        assert ref["makespan"] >= bf["makespan"]
    r50 = nets.fuse_bnrelu(nets.resnet50())
    d = _net_profile(r50, 64, link, 0)
    total = sum(d["bytes"])
    po, pc = both(d, resident=200_000_000, budget=200_000_000 + int(total * 0.35))
    ref = OP.pooch(po, li_cap=3)
    cls, rep = pc.plan("pooch", li_cap=3)
    assert cls == (ref["cls"] if ref["feasible"] else None)


@pytest.mark.parametrize("seed", range(12))
def test_no_host_arena_plans_keep_recompute(seed):
    """A context without a pinned host arena (host budget 1 byte, as make_problem sets it) still
    gets keep / recompute plans (the sink used to stay swap and make every start
    infeasible): the step-1 start keeps the sink (Reading 37), the C++ planner equals the oracle,
    and no map is swapped."""
    d, budget = _tight(seed, 5 + seed % 4)
    po, pc = both(d, resident=10, budget=budget, host_budget=1)
    ref = OP.pooch(po, li_cap=16)
    cls, rep = pc.plan("pooch", threads=2)
    if not ref["feasible"]:
        assert cls is None
        return
    assert cls == ref["cls"] and rep.makespan_ns == ref["makespan"]
    assert OS.SWAP not in cls


def test_no_host_arena_start():
    """The ADVICE r01 case. Without a host arena step 1 starts from the recompute class with the
    sink kept (Reading 37). (a) Four maps computed from the (resident) input: that start fits, so
    PoocH returns it (step 1 only turns swap into keep, so nothing improves on it without a host
    arena) -- C++ = oracle, feasible, no swap. (b) A 6-map chain: recomputing everything replays
    the whole forward at the first backward task, the start runs out of memory and PoocH reports
    infeasible (its precondition, "problem exceeds plannable size"), although brute force
    finds keep / recompute plans -- a documented limit of the paper's search."""
    d = dict(fwd=[10] * 4, bwd=[10] * 4, bytes=[100] * 4, d2h=[5] * 4, h2d=[5] * 4,
             inputs=[[]] * 4, needs=[[0], [1], [2], [3]])
    po, pc = both(d, resident=0, budget=200, host_budget=1)
    cls, rep = pc.plan("pooch", threads=1)
    assert cls == OP.pooch(po)["cls"] == [OS.RECOMPUTE, OS.RECOMPUTE, OS.RECOMPUTE, OS.KEEP]
    assert not OS.simulate(po, cls).oom
    n = 6
    d = dict(fwd=[10] * n, bwd=[10] * n, bytes=[100] * n, d2h=[5] * n, h2d=[5] * n,
             inputs=[[]] + [[i] for i in range(n - 1)], needs=[[0]] + [[i - 1, i] for i in range(1, n)])
    po, pc = both(d, resident=0, budget=500, host_budget=1)
    assert OP.brute_force(po)["cls"] is not None
    assert OP.pooch(po)["cls"] is None and pc.plan("pooch", threads=1)[0] is None


def test_li_cap_out_of_range_is_usage_error():
    d, budget = _tight(0, 6)
    _, pc = both(d, resident=10, budget=budget)
    with pytest.raises(Exception):
        pc.plan("pooch", li_cap=21)


def test_chrome_trace_of_the_fig11_timeline():
    """S:L168 timeline export: complete events, microseconds, one tid per lane."""
    f = json.load(open(os.path.join(G, "fig11_chain.json")))
    _, pc = both(f)
    ev = pc.simulate([OS.SWAP] * 8, events=True)["events"]
    tr = pp.chrome_trace(ev, names=["l%d" % i for i in range(8)])
    assert len(tr) == len(ev) and all(e["ph"] == "X" for e in tr)
    json.loads(json.dumps(tr))
    f7 = [e for e in tr if e["name"] == "fwd l7"][0]
    assert (f7["ts"], f7["dur"], f7["tid"]) == (70e-3, 10e-3, 0)       # F7 = [70, 80] ns
    assert sorted({e["tid"] for e in tr}) == [0, 1, 2]
