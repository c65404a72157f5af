"""Timeline + memory simulator of one out-of-core iteration (oracle, C3).

The paper evaluates a classification by simulating "an execution timeline and
memory management processes" (Sec. 4.1.2) from profiled times
(Sec. 4.2), with the swap-in schedule of Sec. 4.3,
because "it is difficult to formulate the execution time with a simple linear
equation due to pipelined processing and data dependency". This is a
plain event loop written for reading, not speed. The rules, each with its
source (Readings are numbered as in DESIGN.md):

Lanes: COMPUTE, D2H, H2D, one task at a time each (Reading 10).

Shared host link (Reading 51): a copy's profiled time is its duration with
  the other copy lane idle; while both copy lanes are busy the D2H copy
  progresses at duplex_d2h / 1000 and the H2D copy at duplex_h2d / 1000 of
  that rate (the probed duplex over single-direction bandwidth, per mille).
  Work is kept in integer ns x 1000; a copy ends at the first integer ns at
  which its remaining work is <= 0. duplex = 1000 (the default) is the plain
  model in which each copy takes exactly its profiled time.

COMPUTE program: F(0..n-1) in topological order; then for o = n-1..0 the
  recompute tasks bwd(o) needs that are not yet regenerated (recursively,
  P:L114-116 "recomputation recursively"; inputs before outputs), then B(o).

Dependencies (Sec. 3.1): a swap-out of map m starts after F(m) and
  F(c) for every forward consumer c ("must wait for all the forward
  computations that use the data"); B(o) and REC(r) start after every swap
  map they read has been swapped in ("must wait for all the necessary data to
  be swapped in"); a swap-in starts after that map's swap-out.

Memory ledger (Reading 4): resident base R at t=0. Map m is allocated at
  F(m) start. keep: freed at the end of its last use. swap: freed at its
  swap-out end (Reading 5); its swap-in reserves at issue and is
  freed at the end of its last backward-phase use. recompute: freed at the
  end of its last forward use, re-allocated at REC(m) start, freed at the end
  of its last backward-phase use (Reading 6). A map with no backward-phase
  use is freed at the end of its last forward use, whatever its class.
  Gradient g(m) (m not the sink) is allocated at the start of B(c) for the
  first consumer c of m in backward order and freed at the end of B(m).
  A COMPUTE task whose allocation does not fit waits; if no lane can make
  progress the plan is out of memory (reported, not raised).

Swap-in issue (Sec. 4.3): FIFO in need order, no bypass. SuperNeurons
  ("Each swap-in starts simultaneously with the computation of the
  immediately preceding convolution layer"): once the last convolution
  backward task before the map's first user has started. Eager
  ("simply executes swapping-in when there is room"): once every
  forward task has ended. Naive ("each swap-in simply
  starts simultaneously with the previous computation", Reading 8): once the
  program task just before the map's first backward-phase user has started
  (for the first backward task that is the last forward task).
  "Room" (Reading 9): live + bytes(m) + H(m) <= budget, where H(m) is the
  peak extra memory the COMPUTE program needs from its next unstarted task
  up to m's first use ("The amount of free memory at each time of backward
  can be judged from profiling result").

Tie order: completions then starts, each in lane order COMPUTE, D2H, H2D;
  ready swap-outs by (ready time, id).

Outputs: makespan (last task end), peak bytes, OOM flag, per-map swap-in
  stall (excess of the swap-in end over the moment COMPUTE was otherwise free
  to run the first user, Reading 14), L_O = swap-outs ending after the last
  forward task (Reading 13), L_I = maps with stall > 0.
"""
from __future__ import annotations

KEEP, SWAP, RECOMPUTE, FREE = 0, 1, 2, 3   # FREE = zero-byte, zero-transfer keep (Eq. 1 baseline)
EAGER, NAIVE, SN = 0, 1, 2     # SN: swap-in with the preceding convolution (SuperNeurons)


class Profile:
    """Per-task profile: fwd/bwd/recompute ns, map bytes,
    swap-out/in ns, graph (inputs, needs), resident base, budget, tail."""

    def __init__(self, fwd, bwd, nbytes, d2h, h2d, inputs, needs, resident=0,
                 budget=1 << 62, rec=None, tail=0, is_conv=None, host_budget=None,
                 duplex=(1000, 1000)):
        self.n = len(fwd)
        self.fwd, self.bwd, self.bytes = list(fwd), list(bwd), list(nbytes)
        self.d2h, self.h2d = list(d2h), list(h2d)
        self.rec = list(fwd) if rec is None else list(rec)
        self.inputs = [[j for j in ins if j >= 0] for ins in inputs]
        self.needs = [sorted(set(nd)) for nd in needs]
        self.resident, self.budget, self.tail = resident, budget, tail
        self.is_conv = [False] * self.n if is_conv is None else [bool(v) for v in is_conv]
        self.host_budget = host_budget      # pinned host bytes for the swap class (None: unlimited)
        self.duplex_d2h, self.duplex_h2d = int(duplex[0]), int(duplex[1])   # Reading 51
        assert 0 < self.duplex_d2h <= 1000 and 0 < self.duplex_h2d <= 1000
        for i in range(self.n):
            assert all(j < i for j in self.inputs[i]), "inputs must be topological"
            assert self.fwd[i] > 0 and self.bwd[i] > 0 and self.rec[i] > 0
            assert self.d2h[i] > 0 and self.h2d[i] > 0 and self.bytes[i] >= 0

    @staticmethod
    def from_dict(d, **kw):
        if "is_conv" in d and "is_conv" not in kw:
            kw["is_conv"] = d["is_conv"]
        return Profile(d["fwd"], d["bwd"], d["bytes"], d["d2h"], d["h2d"], d["inputs"],
                       d["needs"], **kw)


class Result:
    def __init__(self):
        self.oom = False
        self.makespan = 0
        self.peak = 0
        self.events = []          # (lane, kind, id, start, end)
        self.stall = {}
        self.L_O = set()
        self.L_I = set()
        self.fwd_end = 0


def build_program(p: Profile, cls):
    """COMPUTE lane order: [('F', i)] * n then recompute chains and B(o)."""
    prog = [("F", i) for i in range(p.n)]
    regenerated = set()

    def chain(m):
        for j in p.inputs[m]:
            if cls[j] == RECOMPUTE and j not in regenerated:
                chain(j)
        prog.append(("R", m))
        regenerated.add(m)

    for o in reversed(range(p.n)):
        for m in p.needs[o]:
            if cls[m] == RECOMPUTE and m not in regenerated:
                chain(m)
        prog.append(("B", o))
    return prog


def _reads(p, task):
    kind, i = task
    if kind == "F":
        return list(p.inputs[i])
    if kind == "R":
        return list(p.inputs[i])
    return list(p.needs[i])


def simulate(p: Profile, cls, sched=EAGER, budget=None) -> Result:
    budget = p.budget if budget is None else budget
    n = p.n
    cls = list(cls)
    size = [0 if cls[m] == FREE else p.bytes[m] for m in range(n)]
    prog = build_program(p, cls)
    P = len(prog)
    consumers = [[] for _ in range(n)]
    for c in range(n):
        for m in p.inputs[c]:
            consumers[m].append(c)

    # positions of uses
    last_fwd_use = [max([m] + consumers[m]) for m in range(n)]       # program pos == task id in fwd
    bwd_uses = [[] for _ in range(n)]
    for q in range(n, P):
        for m in _reads(p, prog[q]):
            bwd_uses[m].append(q)
    need = [min(u) if u else None for u in bwd_uses]
    last_bwd = [max(u) if u else None for u in bwd_uses]
    is_swap = [cls[m] == SWAP and need[m] is not None for m in range(n)]

    # allocation A[q] and compute-caused frees Fr[q] per program position
    A = [0] * P
    Fr = [0] * P
    bpos = {prog[q][1]: q for q in range(n, P) if prog[q][0] == "B"}
    for q, (kind, i) in enumerate(prog):
        if kind in ("F", "R"):
            A[q] += size[i]
    for m in range(n):
        if consumers[m]:   # gradient buffer of m
            A[bpos[max(consumers[m])]] += p.bytes[m]
            Fr[bpos[m]] += p.bytes[m]
    for m in range(n):
        c = cls[m]
        if need[m] is None:
            Fr[last_fwd_use[m]] += size[m]
        elif c in (KEEP, FREE):
            Fr[last_bwd[m]] += size[m]
        elif c == SWAP:
            Fr[last_bwd[m]] += size[m]          # swapped-in instance
        else:
            Fr[last_fwd_use[m]] += size[m]      # discard after forward
            Fr[last_bwd[m]] += size[m]          # regenerated instance

    def dur(task):
        kind, i = task
        return p.fwd[i] if kind == "F" else (p.rec[i] if kind == "R" else p.bwd[i])

    fifo = sorted([m for m in range(n) if is_swap[m]], key=lambda m: (need[m], m))
    if p.host_budget is not None and sum(p.bytes[m] for m in fifo) > p.host_budget:
        res = Result()                     # the swap class does not fit the host arena (Reading 36)
        res.oom = True
        return res
    ready_at = [[] for _ in range(n)]          # swap maps whose swap-out may start after F(q)
    for m in range(n):
        if is_swap[m]:
            ready_at[last_fwd_use[m]].append(m)
    res = Result()
    t = 0
    live = p.resident
    peak = live
    pc = 0
    c_run = None          # (q, end)
    start_of = [None] * P
    end_of = [None] * P
    d_run = None          # [m, remaining work (ns x 1000), event index]
    d_ready = {}          # m -> ready time
    out_end = {}
    h_run = None          # [m, remaining work (ns x 1000), event index]
    hq = 0
    in_end = {}
    fwd_done = 0
    fwd_end = None

    def sn_trig(m):
        for q in range(need[m] - 1, n - 1, -1):
            if prog[q][0] == "B" and p.is_conv[prog[q][1]]:
                return q
        return n - 1

    def headroom(m):
        best, acc = 0, 0
        for q in range(pc, need[m] + 1):
            best = max(best, acc + A[q])
            acc += A[q] - Fr[q]
        return best

    while True:
        # ---- completions at t (COMPUTE, D2H, H2D)
        if c_run is not None and c_run[1] == t:
            q = c_run[0]
            end_of[q] = t
            live -= Fr[q]
            c_run = None
            if prog[q][0] == "F":
                fwd_done += 1
                for m in ready_at[q]:
                    d_ready[m] = t
                if fwd_done == n:
                    fwd_end = t
        if d_run is not None and d_run[1] <= 0:
            m = d_run[0]
            live -= size[m]
            out_end[m] = t
            res.events[d_run[2]] = res.events[d_run[2]][:4] + (t,)
            d_run = None
        if h_run is not None and h_run[1] <= 0:
            in_end[h_run[0]] = t
            res.events[h_run[2]] = res.events[h_run[2]][:4] + (t,)
            h_run = None
        # ---- starts at t (COMPUTE, D2H, H2D)
        if c_run is None and pc < P:
            task = prog[pc]
            ok = True
            if task[0] != "F":
                for m in _reads(p, task):
                    if is_swap[m] and (m not in in_end or in_end[m] > t):
                        ok = False
            if ok and live + A[pc] <= budget:
                live += A[pc]
                peak = max(peak, live)
                start_of[pc] = t
                c_run = (pc, t + dur(task))
                res.events.append(("COMPUTE", task[0], task[1], t, t + dur(task)))
                pc += 1
        if d_run is None and d_ready:
            m = min(d_ready, key=lambda k: (d_ready[k], k))
            del d_ready[m]
            d_run = [m, 1000 * p.d2h[m], len(res.events)]
            res.events.append(("D2H", "O", m, t, None))     # end set at completion
        if h_run is None and hq < len(fifo):
            m = fifo[hq]
            if sched == EAGER:
                phase_ok = fwd_end is not None and fwd_end <= t
            else:
                trig = need[m] - 1
                if sched == SN:     # the backward task of the preceding convolution layer
                    trig = sn_trig(m)
                phase_ok = start_of[trig] is not None and start_of[trig] <= t
            if phase_ok and m in out_end and out_end[m] <= t and \
                    live + size[m] + headroom(m) <= budget:
                live += size[m]
                peak = max(peak, live)
                h_run = [m, 1000 * p.h2d[m], len(res.events)]
                res.events.append(("H2D", "I", m, t, None))
                hq += 1
        # ---- advance (copy rates: Reading 51)
        both = d_run is not None and h_run is not None
        rd = p.duplex_d2h if both else 1000
        rh = p.duplex_h2d if both else 1000
        ends = []
        if c_run is not None:
            ends.append(c_run[1])
        if d_run is not None:
            ends.append(t + -(-d_run[1] // rd))       # ceil(remaining / rate)
        if h_run is not None:
            ends.append(t + -(-h_run[1] // rh))
        if not ends:
            if pc < P or hq < len(fifo) or d_ready:
                res.oom = True
            break
        t_next = min(ends)
        if d_run is not None:
            d_run[1] -= (t_next - t) * rd
        if h_run is not None:
            h_run[1] -= (t_next - t) * rh
        t = t_next

    res.peak = peak
    if res.oom:
        return res
    res.makespan = max(e[4] for e in res.events)
    res.fwd_end = fwd_end
    for m in fifo:
        q = need[m]
        lane_ready = end_of[q - 1]
        res.stall[m] = max(0, in_end[m] - lane_ready)
    res.L_O = {m for m in range(n) if is_swap[m] and out_end[m] > fwd_end}
    res.L_I = {m for m, s in res.stall.items() if s > 0}
    return res


def makespan(p, cls, sched=EAGER):
    r = simulate(p, cls, sched)
    return None if r.oom else r.makespan
