"""What-if: plan a measured ResNet-50 profile with and without BN-ReLU prologue fusion.

Usage: python tools/f2_whatif.py gpurun_out/profile_cfg2.json [conv_slowdown]

The fused graph drops every BN-ReLU map whose only consumer is a conv (the conv applies
relu(bn(c)) to its operand on load): the conv's input becomes c, its backward also runs the
BN-ReLU backward. Times come from the measured (unfused) profile; the fused conv's forward is
scaled by ``conv_slowdown`` (default 1.0).
"""
import json
import sys

sys.path.insert(0, ".")
from oracle import nets  # noqa: E402  (graph only: inputs / needs / kinds)
from paper_1907_05013_b200.planning import PlanProblem  # noqa: E402

d = json.load(open(sys.argv[1]))
slow = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
pr = d["profile"]
net = nets.resnet50()
n = len(net.tasks)
inputs = [[j for j in t.inputs if j >= 0] for t in net.tasks]
needs = [net.needs(i) for i in range(n)]
consumers = [[k for k in range(n) if i in inputs[k]] for i in range(n)]
budget = d["budget"]
resident = pr["resident"]


def plan(fwd, bwd, rec, nbytes, d2h, h2d, ins, nds, is_conv):
    p = PlanProblem(fwd, bwd, nbytes, d2h, h2d, ins, nds, resident=resident, budget=budget, rec=rec,
                    tail=pr["tail"], is_conv=is_conv)
    cls, rep = p.plan("pooch", li_cap=12)
    inc = p.simulate([0] * len(fwd))
    return cls, rep, inc


is_conv = [int(t.kind == "conv") for t in net.tasks]
cls, rep, inc = plan(pr["fwd"], pr["bwd"], pr["rec"], pr["bytes"], pr["d2h"], pr["h2d"], inputs, needs, is_conv)
print("unfused: %d maps, %.1f GB, plan k/s/r = %d/%d/%d, makespan %.1f ms (in-core sim %.1f ms, oom=%s)" % (
    n, sum(pr["bytes"]) / 1e9, cls.count(0), cls.count(1), cls.count(2), rep.makespan_ns / 1e6,
    inc["makespan"] / 1e6, inc["oom"]))

fused = {i for i, t in enumerate(net.tasks) if t.kind == "bnrelu" and len(consumers[i]) == 1
         and net.tasks[consumers[i][0]].kind == "conv" and inputs[consumers[i][0]] == [i]}
keep = [i for i in range(n) if i not in fused]
new_id = {o: k for k, o in enumerate(keep)}


def remap(lst):
    out = []
    for j in lst:
        j = inputs[j][0] if j in fused else j
        out.append(new_id[j])
    return sorted(set(out))


F, Bw, R, NB, D, H, I, N, C = [], [], [], [], [], [], [], [], []
for o in keep:
    f, b = pr["fwd"][o], pr["bwd"][o]
    if net.tasks[o].kind == "conv" and inputs[o] and inputs[o][0] in fused:
        r = inputs[o][0]
        f = int(f * slow)
        b = b + pr["bwd"][r]
    F.append(f)
    Bw.append(b)
    R.append(f if net.tasks[o].kind == "conv" else pr["rec"][o])
    NB.append(pr["bytes"][o])
    D.append(pr["d2h"][o])
    H.append(pr["h2d"][o])
    I.append(remap(inputs[o]))
    N.append(remap(needs[o]))
    C.append(is_conv[o])
cls2, rep2, inc2 = plan(F, Bw, R, NB, D, H, I, N, C)
print("fused  : %d maps, %.1f GB, plan k/s/r = %d/%d/%d, makespan %.1f ms (in-core sim %.1f ms, oom=%s)" % (
    len(keep), sum(NB) / 1e9, cls2.count(0), cls2.count(1), cls2.count(2), rep2.makespan_ns / 1e6,
    inc2["makespan"] / 1e6, inc2["oom"]))
