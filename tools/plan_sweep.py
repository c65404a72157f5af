"""Offline: re-plan a measured profile (bench.py --dump-profile) with the C++ planner at several
li_cap values and strategies; prints predicted makespans and planner cost.

Usage: python tools/plan_sweep.py gpurun_out/profile_cfg2.json
"""
import json
import sys
import time

sys.path.insert(0, ".")
from oracle import nets  # noqa: E402  (graph only)
from paper_1907_05013_b200.planning import PlanProblem  # noqa: E402

d = json.load(open(sys.argv[1]))
pr = d["profile"]
net = nets.resnet50()
n = len(net.tasks)
inputs = [[j for j in t.inputs if j >= 0] for t in net.tasks]
needs = [net.needs(i) for i in range(n)]
is_conv = [int(t.kind == "conv") for t in net.tasks]
p = PlanProblem(pr["fwd"], pr["bwd"], pr["bytes"], pr["d2h"], pr["h2d"], inputs, needs, resident=pr["resident"],
                budget=d["budget"], rec=pr["rec"], tail=pr["tail"], is_conv=is_conv)
print("measured plan (bench): k/s/r = %d/%d/%d" % (d["classes"].count(0), d["classes"].count(1), d["classes"].count(2)),
      "sim %.1f ms" % (p.simulate(d["classes"])["makespan"] / 1e6))
for strat in ("swap_all", "swap_opt", "superneurons"):
    cls, rep = p.plan(strat)
    print("%-14s %s" % (strat, "infeasible" if cls is None else "%.1f ms" % (rep.makespan_ns / 1e6)))
for cap in (4, 8, 10, 12, 14, 16):
    t0 = time.time()
    cls, rep = p.plan("pooch", li_cap=cap)
    print("pooch li_cap=%2d: %.1f ms  k/s/r = %d/%d/%d  sims %d  %.1f s" % (
        cap, rep.makespan_ns / 1e6, cls.count(0), cls.count(1), cls.count(2), rep.n_sims, time.time() - t0))
