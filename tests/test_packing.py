"""Static offset packing (row a6): buffer instances that are live at the same time
never share bytes, and the packed high-water mark stays within the capacity."""
import pytest

import synthdata
from oracle import nets
from oracle.sim import KEEP, RECOMPUTE, SWAP, Profile, simulate

pp = pytest.importorskip("paper_1907_05013_b200.planning")


def _check(res, cap):
    live = [b for b in range(len(res["offsets"])) if res["alloc"][b] >= 0]
    assert res["high_water"] <= cap
    for i, a in enumerate(live):
        a0, a1 = int(res["alloc"][a]), int(res["free"][a]) if res["free"][a] >= 0 else 1 << 30
        ra = (int(res["offsets"][a]), int(res["offsets"][a]) + int(res["sizes"][a]))
        assert ra[1] <= cap
        for b in live[i + 1:]:
            b0, b1 = int(res["alloc"][b]), int(res["free"][b]) if res["free"][b] >= 0 else 1 << 30
            if a0 < b1 and b0 < a1:                          # lifetimes overlap in the ledger
                rb = (int(res["offsets"][b]), int(res["offsets"][b]) + int(res["sizes"][b]))
                assert ra[1] <= rb[0] or rb[1] <= ra[0], (a, b, ra, rb)


@pytest.mark.parametrize("seed", range(30))
def test_random_plans_pack_without_overlap(seed):
    g = synthdata.rng(3000 + seed)
    n = int(g.integers(2, 12))
    d = synthdata.random_profile(n, seed, dag=seed % 2 == 0, max_bytes=4096)
    budget = int(sum(d["bytes"]) * 2)
    pc = pp.PlanProblem.from_dict(d, resident=0, budget=budget)
    for _ in range(5):
        cls = [int(c) for c in g.integers(0, 3, n)]
        cls[-1] = min(cls[-1], SWAP)
        r = pc.simulate(cls)
        if r["oom"]:
            continue
        res = pc.pack(cls, 4 * budget)
        assert res is not None
        _check(res, 4 * budget)


def test_resnet50_pooch_plan_packs_under_budget():
    net = nets.resnet50()
    n = len(net.tasks)
    nbytes = [640 * net.map_bytes_per_image(i) for i in range(n)]
    fwd = [max(1, b // 6000) for b in nbytes]
    x = [max(1, b // 55) for b in nbytes]
    inputs = [[j for j in t.inputs if j >= 0] for t in net.tasks]
    needs = [net.needs(i) for i in range(n)]
    budget = 15 << 30
    pc = pp.PlanProblem(fwd, [2 * f for f in fwd], nbytes, x, x, inputs, needs, resident=0, budget=budget)
    # the executor's rule (pooch_plan): if best-fit fragments, plan against 2% less and retry
    for attempt in range(12):
        b_k = budget - attempt * (budget // 50)
        cls, rep = pp.PlanProblem(fwd, [2 * f for f in fwd], nbytes, x, x, inputs, needs, resident=0,
                                  budget=b_k).plan("pooch", li_cap=8)
        assert cls is not None
        res = pc.pack(cls, budget)
        if res is not None:
            break
    assert res is not None, "no packable plan after 12 attempts"
    _check(res, budget)
