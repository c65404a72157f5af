"""Pins for the oracle simulator (C3): SPEC hand traces, the paper's Fig. 11
stall sets, and timeline invariants."""
import json
import os

import pytest

import synthdata
from oracle import sim
from oracle.sim import EAGER, FREE, KEEP, NAIVE, RECOMPUTE, SWAP, Profile, simulate

G = os.path.join(os.path.dirname(__file__), "golden")


def test_spec_hand_traces():
    d = json.load(open(os.path.join(G, "spec_traces.json")))
    p = Profile.from_dict(d["profile"])
    assert simulate(p, [KEEP]).makespan == d["keep_makespan"]
    r = simulate(p, [SWAP])
    assert [list(e) for e in r.events] == d["swap_events"]
    assert r.makespan == d["swap_makespan"]
    assert r.makespan - simulate(p, [FREE]).makespan == d["swap_overhead"]


def test_fig11_stall_sets():
    d = json.load(open(os.path.join(G, "fig11_chain.json")))
    p = Profile.from_dict(d)
    r = simulate(p, [SWAP] * 8)
    assert sorted(r.L_O) == d["L_O"]
    assert sorted(r.L_I) == d["L_I"]
    assert sorted(r.L_O - r.L_I) == d["L_O_minus_L_I"]


def _check_invariants(p, cls, r, budget):
    by_lane = {}
    for lane, kind, i, s, e in r.events:
        by_lane.setdefault(lane, []).append((s, e, kind, i))
        dur = {"F": p.fwd[i], "B": p.bwd[i], "R": p.rec[i], "O": p.d2h[i], "I": p.h2d[i]}[kind]
        assert e - s == dur                                   # duration exactness
    for lane, evs in by_lane.items():                         # lane exclusivity
        evs.sort()
        for a, b in zip(evs, evs[1:]):
            assert a[1] <= b[0]
    F = {i: (s, e) for lane, k, i, s, e in r.events if k == "F"}
    O = {i: (s, e) for lane, k, i, s, e in r.events if k == "O"}
    I = {i: (s, e) for lane, k, i, s, e in r.events if k == "I"}
    for m, (s, e) in O.items():                               # swap-out after all fwd users
        assert s >= F[m][1]
        for c in range(p.n):
            if m in p.inputs[c]:
                assert s >= F[c][1]
    for m, (s, e) in I.items():
        assert s >= O[m][1]
    for lane, k, i, s, e in r.events:                         # bwd after its swap-ins
        if k in ("B", "R"):
            reads = p.needs[i] if k == "B" else p.inputs[i]
            for m in reads:
                if cls[m] == SWAP:
                    assert I[m][1] <= s
    assert r.peak <= budget
    assert r.makespan == max(e for *_, e in r.events)


@pytest.mark.parametrize("seed", range(40))
def test_invariants_random(seed):
    d = synthdata.random_profile(6, seed, dag=seed % 2 == 1)
    g = synthdata.rng(seed)
    budget = int(sum(d["bytes"]) * g.uniform(0.4, 1.5)) + 10
    p = Profile.from_dict(d, resident=10, budget=budget)
    for trial in range(6):
        cls = [int(c) for c in g.integers(0, 3, 6)]
        cls[-1] = min(cls[-1], SWAP)
        for sched in (EAGER, NAIVE):
            r = simulate(p, cls, sched)
            if not r.oom:
                _check_invariants(p, cls, r, budget)
            r2 = simulate(p, cls, sched)                      # determinism
            assert (r.oom, r.makespan, r.peak, r.events) == (r2.oom, r2.makespan, r2.peak, r2.events)


@pytest.mark.parametrize("seed", range(20))
def test_all_keep_chain_is_sum_of_compute(seed):
    d = synthdata.random_profile(7, seed)
    p = Profile.from_dict(d)
    r = simulate(p, [KEEP] * 7)
    assert r.makespan == sum(d["fwd"]) + sum(d["bwd"])


@pytest.mark.parametrize("seed", range(20))
def test_eager_not_slower_than_naive_with_ample_memory(seed):
    d = synthdata.random_profile(8, seed)
    p = Profile.from_dict(d)
    assert simulate(p, [SWAP] * 8, EAGER).makespan <= simulate(p, [SWAP] * 8, NAIVE).makespan


def test_recompute_chain_program():
    # 2-chain A->B with A recompute; 3-chain A,B recompute, C keep
    d = synthdata.random_profile(3, 0)
    p = Profile.from_dict(d)
    prog = sim.build_program(p, [RECOMPUTE, RECOMPUTE, KEEP])
    bwd = prog[3:]
    # B(2) needs maps 1,2 -> chain R(0), R(1) (recursive, inputs first) before B(2)
    assert bwd[:3] == [("R", 0), ("R", 1), ("B", 2)]
    assert bwd[3:] == [("B", 1), ("B", 0)]


def test_oom_reported_not_raised():
    d = synthdata.random_profile(4, 1)
    p = Profile.from_dict(d, resident=5, budget=5 + max(d["bytes"]) - 1)
    assert simulate(p, [SWAP] * 4).oom
