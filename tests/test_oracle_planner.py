"""Pins for the oracle planners (C4): brute force is the optimum under the
cost model; PoocH is feasible, no better than it, and obeys the paper's
ordering claims."""
import pytest

import synthdata
from oracle import planner
from oracle.sim import EAGER, KEEP, NAIVE, RECOMPUTE, SWAP, Profile, simulate


def _tight(seed, n=6, dag=False, frac=None):
    d = synthdata.random_profile(n, seed, dag=dag)
    g = synthdata.rng(77 + seed)
    frac = g.uniform(0.45, 0.9) if frac is None else frac
    budget = 10 + max(3 * max(d["bytes"]), int(sum(d["bytes"]) * frac))
    return Profile.from_dict(d, resident=10, budget=budget)


def test_spec_exhaustive_examples():
    p = Profile([4], [4], [8], [6], [6], [[]], [[0]], resident=0, budget=100)
    assert planner.brute_force(p)["cls"] == [KEEP]
    p = Profile([4], [4], [8], [6], [6], [[]], [[0]], resident=4, budget=11)
    r = planner.brute_force(p)
    assert r["cls"] is None                 # needs 8 bytes on top of 4 at fwd: infeasible
    p = Profile([4, 4], [4, 4], [8, 8], [1, 1], [1, 1], [[], [0]], [[0], [0, 1]], resident=0, budget=16)
    assert planner.brute_force(p)["evaluated"] == 2 * 3


@pytest.mark.parametrize("seed", range(20))
def test_pooch_feasible_and_not_below_optimum(seed):
    p = _tight(seed, dag=seed % 3 == 0)
    bf = planner.brute_force(p)
    po = planner.pooch(p)
    if bf["cls"] is None:
        assert not po["feasible"] or simulate(p, po["cls"]).oom is False
        return
    if not po["feasible"]:
        # PoocH starts from all-swap; it may be infeasible where another plan fits
        assert simulate(p, [SWAP] * p.n).oom
        return
    r = simulate(p, po["cls"])
    assert not r.oom and r.peak <= p.budget
    assert r.makespan == po["makespan"]
    assert po["makespan"] >= bf["makespan"]
    assert po["cls"][-1] != RECOMPUTE


@pytest.mark.parametrize("seed", range(20))
def test_monotone_chain(seed):
    p = _tight(seed, n=8)
    if simulate(p, [SWAP] * p.n).oom:
        pytest.skip("all-swap infeasible")
    s = planner.strategies(p)
    assert s["pooch"] <= s["swap_opt"] <= s["swap_all"]


@pytest.mark.parametrize("seed", range(10))
def test_incore_fixpoint(seed):
    d = synthdata.random_profile(6, seed)
    p = Profile.from_dict(d, resident=0, budget=10 * sum(d["bytes"]))
    po = planner.pooch(p)
    assert po["cls"] == [KEEP] * 6 and po["makespan"] == sum(d["fwd"]) + sum(d["bwd"])


@pytest.mark.parametrize("seed", range(10))
def test_step2_commits_only_r_below_one(seed):
    p = _tight(seed, n=8)
    log = []
    po = planner.pooch(p, log=log)
    for entry in log:
        if entry[0] == "commit":
            assert entry[2] < 1.0


def test_zero_cost_replay_goes_recompute_and_hidden_swap_stays():
    # Eq. (1) limits: X=map 0 replays in 1 ns from the resident
    # input but its 50 ns transfers stall; map 1 (the sink) can't recompute.
    p = Profile([1, 40], [40, 40], [4, 4], [50, 1], [50, 1], [[], [0]], [[0], [0, 1]],
                resident=0, budget=12)
    cls, ms, _ = planner.step2(p, [SWAP, SWAP])
    assert cls == [RECOMPUTE, SWAP]


def test_slower_link_more_recompute():
    """Table 3 direction: the slower link yields more recompute."""
    counts = []
    for scale in (1, 5):              # scale = link slowness
        d = synthdata.random_profile(10, 3, max_x=10)
        d["fwd"] = [2 if i % 2 else 30 for i in range(10)]      # cheap BN-like layers interleaved
        d["d2h"] = [v * scale for v in [12] * 10]
        d["h2d"] = [v * scale for v in [12] * 10]
        d["bytes"] = [8] * 10
        p = Profile.from_dict(d, resident=0, budget=40)
        po = planner.pooch(p)
        counts.append(po["cls"].count(RECOMPUTE))
    assert counts[1] > counts[0]
