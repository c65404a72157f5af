"""What-if: plan a measured ResNet-50 profile with and without BN-ReLU prologue fusion,
through the executor's plan selection (PoocH over a (budget, L_I cap) grid, keep the fastest plan
whose ledger packs into the arena -- DESIGN.md Reading 40).

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
cap = d["budget"] - pr["resident"]


def select(fwd, bwd, rec, nbytes, d2h, h2d, ins, nds, is_conv, li_cap=12):
    best, first = None, None
    for step in range(40):
        b = cap - step * (cap // 250)
        p = PlanProblem(fwd, bwd, nbytes, d2h, h2d, ins, nds, resident=0, budget=b, rec=rec, tail=pr["tail"],
                        is_conv=is_conv)
        for lc in range(4, li_cap + 1, 2):
            cls, rep = p.plan("pooch", li_cap=lc)
            if cls is None or (best is not None and rep.makespan_ns >= best[0]):
                continue
            if p.pack(cls, cap) is not None:
                best = (rep.makespan_ns, cls, b, lc)
                first = step if first is None else first
        if first is not None and step >= first + 4:
            break
    return best


is_conv = [int(t.kind == "conv") for t in net.tasks]
b0 = select(pr["fwd"], pr["bwd"], pr["rec"], pr["bytes"], pr["d2h"], pr["h2d"], inputs, needs, is_conv)
print("unfused: %d maps, %.1f GB, plan k/s/r = %d/%d/%d, makespan %.1f ms (budget %.2f GB, cap %d)" % (
    n, sum(pr["bytes"]) / 1e9, b0[1].count(0), b0[1].count(1), b0[1].count(2), b0[0] / 1e6, b0[2] / 1e9, b0[3]))

fused = {i for i, t in enumerate(net.tasks) if t.kind == "bnrelu" and len(consumers[i]) == 1
         and net.tasks[consumers[i][0]].kind == "conv" and inputs[consumers[i][0]] == [i]}
keep = [i for i in range(n) if i not in fused]
new_id = {o: k for k, o in enumerate(keep)}


def remap(lst):
    return sorted({new_id[inputs[j][0] if j in fused else j] for j in lst})


F, Bw, R, NB, D, H, I, N, C = [], [], [], [], [], [], [], [], []
for o in keep:
    f, b = pr["fwd"][o], pr["bwd"][o]
    if net.tasks[o].kind == "conv" and inputs[o] and inputs[o][0] in fused:
        f = int(f * slow)
        b = b + pr["bwd"][inputs[o][0]]
    F.append(f)
    Bw.append(b)
    R.append(f if net.tasks[o].kind == "conv" else pr["rec"][o])
    NB.append(pr["bytes"][o])
    D.append(pr["d2h"][o])
    H.append(pr["h2d"][o])
    I.append(remap(inputs[o]))
    N.append(remap(needs[o]))
    C.append(is_conv[o])
b1 = select(F, Bw, R, NB, D, H, I, N, C)
print("fused  : %d maps, %.1f GB, plan k/s/r = %d/%d/%d, makespan %.1f ms (budget %.2f GB, cap %d)" % (
    len(keep), sum(NB) / 1e9, b1[1].count(0), b1[1].count(1), b1[1].count(2), b1[0] / 1e6, b1[2] / 1e9, b1[3]))
