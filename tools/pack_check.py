"""Offline: the executor's plan -> pack loop (pooch_plan) on a measured profile: plan against the
budget, pack the simulated ledger into the arena, and on fragmentation re-plan 2 % lower.
Usage: python tools/pack_check.py gpurun_out/profile_cfg2.json [li_cap]"""
import json
import sys

sys.path.insert(0, ".")
from oracle import nets  # noqa: E402  (graph only)
from paper_1907_05013_b200.planning import PlanProblem  # noqa: E402

d = json.load(open(sys.argv[1]))
cap_li = int(sys.argv[2]) if len(sys.argv) > 2 else 12
pr = d["profile"]
net = nets.resnet50()
n = len(net.tasks)
inputs = [[j for j in t.inputs if j >= 0] for t in net.tasks]
needs = [net.needs(i) for i in range(n)]
is_conv = [int(t.kind == "conv") for t in net.tasks]
cap = d["budget"] - pr["resident"]
for attempt in range(12):
    b = cap - attempt * (cap // 50)
    p = PlanProblem(pr["fwd"], pr["bwd"], pr["bytes"], pr["d2h"], pr["h2d"], inputs, needs, resident=0, budget=b,
                    rec=pr["rec"], tail=pr["tail"], is_conv=is_conv)
    cls, rep = p.plan("pooch", li_cap=cap_li)
    sim = p.simulate(cls)
    res = p.pack(cls, cap)
    print("attempt %d budget %.2f GB: makespan %.1f ms, sim peak %.2f GB, packed %s" % (
        attempt, b / 1e9, rep.makespan_ns / 1e6, sim["peak"] / 1e9,
        "%.2f GB" % (res["high_water"] / 1e9) if res is not None else "FAILED"))
    if res is not None:
        break
print("fragmentation (packed high-water with unlimited capacity / simulated peak):")
for attempt in range(5):
    b = cap - attempt * (cap // 50)
    p = PlanProblem(pr["fwd"], pr["bwd"], pr["bytes"], pr["d2h"], pr["h2d"], inputs, needs, resident=0, budget=b,
                    rec=pr["rec"], tail=pr["tail"], is_conv=is_conv)
    cls, rep = p.plan("pooch", li_cap=cap_li)
    sim = p.simulate(cls)
    res = p.pack(cls, 1 << 50)
    print("  budget %.2f GB: peak %.3f GB, packed %.3f GB (+%.1f %%)" % (b / 1e9, sim["peak"] / 1e9,
          res["high_water"] / 1e9, 100 * (res["high_water"] / sim["peak"] - 1)))
