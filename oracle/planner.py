"""Keep / swap / recompute classification (oracle, C4). TEST INFRASTRUCTURE ONLY.

Two independent planners over the simulator in ``oracle.sim``:

* ``brute_force`` -- every classification (the O(3^n) search the paper avoids,
  P:L211, Sec. 4.4.1); the sink map is never recompute, so 2*3^(n-1)
  candidates. Feasible minimum by (makespan, #keep, class vector).
* ``pooch`` -- the paper's two-step heuristic, step by step:
  (0) all-keep if it fits (in-core);
  (1) simulate all-swap with eager swap-in ("The safest
      classification ... classifies all feature maps into swap"); OOM ->
      infeasible;
  (2) maps outside L_O u L_I are fixed to swap ("these feature maps are
      classified into swap immediately");
  (3) "a binary search tree, each of whose level corresponds to an element in
      L_I", capped at li_cap members by stall rank (Reading 16); the
      scan set is L_O \\ L_I (plus the cap overflow), from the output layer
      ("in order from the output layer");
  (4) at each leaf "scan elements in L_O \\ L_I linearly and switch a feature
      map from swap to keep, and evaluate the entire classification by
      simulating": a flip that runs out of memory is reverted,
      every other state is recorded (Reading 15);
  (5) the recorded state with minimal makespan;
  (6) step 2, Eq. (1): L = swap maps; each round evaluate
      r(X) = recompute_overhead(X) / swap_overhead(X) for X in L, with both
      overheads measured against the makespan with X free of cost (Reading 17);
      drop every X with r >= 1 (stays swap); stop if L is empty; else move the
      X with the smallest r to recompute (ties: larger bytes, smaller id,
      Reading 19) and repeat.
"""
from __future__ import annotations

import itertools
import math

from .sim import EAGER, FREE, KEEP, NAIVE, RECOMPUTE, SN, SWAP, simulate

INF = math.inf


def _key(ms, cls):
    return (ms, sum(1 for c in cls if c == KEEP), tuple(cls))


def brute_force(p, sched=EAGER, max_n=12):
    """Feasible optimum over all classifications (tiny nets only)."""
    n = p.n
    if n > max_n:
        raise ValueError("brute force guarded to n <= %d" % max_n)
    best = None
    evaluated = infeasible = 0
    for head in itertools.product((KEEP, SWAP, RECOMPUTE), repeat=n - 1):
        for sink in (KEEP, SWAP):
            cls = list(head) + [sink]
            evaluated += 1
            r = simulate(p, cls, sched)
            if r.oom:
                infeasible += 1
                continue
            k = _key(r.makespan, cls)
            if best is None or k < best:
                best = k
    return dict(cls=None if best is None else list(best[2]),
                makespan=None if best is None else best[0],
                evaluated=evaluated, infeasible=infeasible)


def _ms(p, cls, sched=EAGER):
    r = simulate(p, cls, sched)
    return INF if r.oom else r.makespan


def host_fit_base(p):
    """Step 1's starting point. The paper starts from all-swap; when the swap class
    of all-swap exceeds the pinned host arena (Reading 37) the swap maps with the cheapest
    replay per byte (recompute time / bytes; ties: larger bytes, smaller id; never the sink)
    move to recompute until the swap class fits. The sink is never recompute; if it
    alone still does not fit (e.g. no host arena at all), it is kept."""
    n = p.n
    cls = [SWAP] * n
    if p.host_budget is None:
        return cls
    total = sum(p.bytes)
    order = sorted(range(n - 1), key=lambda m: (p.rec[m] / max(p.bytes[m], 1), -p.bytes[m], m))
    for m in order:
        if total <= p.host_budget:
            break
        cls[m] = RECOMPUTE
        total -= p.bytes[m]
    if total > p.host_budget:
        cls[n - 1] = KEEP
    return cls


def step1(p, li_cap=16, sched=EAGER, log=None, trace=None):
    """Keep/swap search (Sec. 4.4.2). Returns (cls, makespan, n_sims). ``trace`` (a list)
    receives every simulated state in evaluation order as (class tuple, makespan or None
    when it ran out of memory) -- the start first, then per leaf the leaf and its scan."""
    n = p.n
    start = host_fit_base(p)
    base = simulate(p, start, sched)
    if base.oom:
        return None, INF, 1
    sims = 1
    if trace is not None:
        trace.append((tuple(start), base.makespan))
    L_O, L_I = set(base.L_O), set(base.L_I)
    ranked = sorted(L_I, key=lambda m: (-base.stall[m], m))
    tree = sorted(ranked[:li_cap])
    overflow = ranked[li_cap:]
    scan = sorted((L_O - set(tree)) | set(overflow), reverse=True)
    best = _key(base.makespan, start)
    for leaf in range(1 << len(tree)):
        cls = list(start)
        for b, m in enumerate(tree):
            if leaf >> b & 1:
                cls[m] = KEEP
        ms = _ms(p, cls, sched)
        sims += 1
        if trace is not None:
            trace.append((tuple(cls), None if ms == INF else ms))
        if ms < INF:
            best = min(best, _key(ms, cls))
        for m in scan:
            cls[m] = KEEP
            ms2 = _ms(p, cls, sched)
            sims += 1
            if trace is not None:
                trace.append((tuple(cls), None if ms2 == INF else ms2))
            if ms2 == INF:
                cls[m] = SWAP          # out of memory: revert, continue the scan
                continue
            best = min(best, _key(ms2, cls))
    if log is not None:
        log.append(("step1", sorted(L_O), sorted(L_I), tree, scan, best[0]))
    return list(best[2]), best[0], sims


def step2(p, cls, sched=EAGER, log=None):
    """Recompute search, Eq. (1) (Sec. 4.4.3). Returns (cls, makespan, n_sims)."""
    n = p.n
    cls = list(cls)
    sink = n - 1
    L = [m for m in range(n) if cls[m] == SWAP and m != sink]
    sims = 0
    t_swap = _ms(p, cls, sched)
    sims += 1
    while L:
        evals = []
        for X in L:
            c0 = list(cls); c0[X] = FREE
            cr = list(cls); cr[X] = RECOMPUTE
            t0 = _ms(p, c0, sched)
            tr = _ms(p, cr, sched)
            sims += 2
            swap_ov = max(0, t_swap - t0)
            rec_ov = INF if tr == INF else max(0, tr - t0)
            r = INF if swap_ov == 0 else rec_ov / swap_ov
            evals.append((r, X, tr))
        keep_going = [(r, X, tr) for (r, X, tr) in evals if r < 1.0]
        if log is not None:
            log.append(("round", [(X, r) for (r, X, _) in evals]))
        if not keep_going:
            break
        r, X, tr = min(keep_going, key=lambda e: (e[0], -p.bytes[e[1]], e[1]))
        cls[X] = RECOMPUTE
        t_swap = tr
        L = [m for (rr, m, _) in keep_going if m != X]
        if log is not None:
            log.append(("commit", X, r, tr))
    return cls, t_swap, sims


def pooch(p, li_cap=16, sched=EAGER, log=None):
    """The full PoocH classification (Sec. 4.4). Returns dict with cls,
    makespan (INF if infeasible) and the number of simulations."""
    n = p.n
    allkeep = simulate(p, [KEEP] * n, sched)
    if not allkeep.oom:
        return dict(cls=[KEEP] * n, makespan=allkeep.makespan, sims=1, feasible=True)
    c1, ms1, s1 = step1(p, li_cap, sched, log)
    if c1 is None:
        return dict(cls=None, makespan=INF, sims=1 + s1, feasible=False)
    c2, ms2, s2 = step2(p, c1, sched, log)
    return dict(cls=c2, makespan=ms2, sims=1 + s1 + s2, feasible=True, swap_opt=c1,
                swap_opt_makespan=ms1)


def superneurons(p):
    """SuperNeurons' static hybrid rule as the paper describes it (Sec. 5.2):
    "Feature maps are stored on GPU memory preferentially from output layer" (keep from the
    sink down while resident + kept bytes fit the budget); "Among the feature maps
    that do not fit ... the feature maps of convolution layer are targets of swapping. The
    feature maps of layers with other types are recomputed"; swap-ins use the SN schedule.
    Returns (cls, makespan or INF)."""
    n = p.n
    cls = [None] * n
    kept = p.resident
    for m in reversed(range(n)):
        if kept + p.bytes[m] > p.budget:
            break
        cls[m] = KEEP
        kept += p.bytes[m]
    for m in range(n):
        if cls[m] is None:
            cls[m] = SWAP if (p.is_conv[m] or m == n - 1) else RECOMPUTE
    return cls, _ms(p, cls, SN)


def strategies(p, li_cap=16):
    """Makespans of the paper's comparison strategies (Sec. 5.1)."""
    n = p.n
    out = {}
    out["incore"] = _ms(p, [KEEP] * n)
    out["swap_all_naive"] = _ms(p, [SWAP] * n, NAIVE)
    out["swap_all"] = _ms(p, [SWAP] * n, EAGER)
    c1, ms1, _ = step1(p, li_cap)
    out["swap_opt"] = ms1
    res = pooch(p, li_cap)
    out["pooch"] = res["makespan"]
    out["superneurons"] = superneurons(p)[1]
    return out
