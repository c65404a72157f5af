"""Host-only planning through the C ABI: pooch_simulate / pooch_plan_problem.

Marshalling only -- the simulator (Sec. 4.1.2) and the PoocH search (Sec. 4.4)
run in libpooch.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import P, PlanReport, Problem, SearchCfg, SimResult, check, lib

KEEP, SWAP, RECOMPUTE, FREE = 0, 1, 2, 3
EAGER, NAIVE, SN = 0, 1, 2
STRATEGIES = {"pooch": 0, "incore": 1, "swap_all_naive": 2, "swap_all": 3, "swap_opt": 4,
              "superneurons": 5, "exhaustive": 6, "fixed": 7}


def _csr(lists):
    ptr = np.zeros(len(lists) + 1, np.int32)
    for i, l in enumerate(lists):
        ptr[i + 1] = ptr[i] + len(l)
    idx = np.array([j for l in lists for j in l] or [0], np.int32)
    return ptr, idx


class PlanProblem:
    """Owns the arrays a pooch_problem points at."""

    def __init__(self, fwd, bwd, nbytes, d2h, h2d, inputs, needs, resident=0, budget=(1 << 62),
                 rec=None, tail=0, is_conv=None, host_budget=None, duplex=(1000, 1000)):
        self.n = len(fwd)
        self._a = {
            "fwd": np.asarray(fwd, np.int64), "bwd": np.asarray(bwd, np.int64),
            "rec": np.asarray(fwd if rec is None else rec, np.int64),
            "d2h": np.asarray(d2h, np.int64), "h2d": np.asarray(h2d, np.int64),
            "bytes": np.asarray(nbytes, np.uint64),
            "is_conv": np.asarray([0] * len(fwd) if is_conv is None else is_conv, np.uint8),
        }
        self._a["in_ptr"], self._a["in_idx"] = _csr([[j for j in l if j >= 0] for l in inputs])
        self._a["need_ptr"], self._a["need_idx"] = _csr(needs)
        a = self._a
        self.c = Problem(self.n, a["fwd"].ctypes.data_as(P(C.c_int64)), a["bwd"].ctypes.data_as(P(C.c_int64)),
                         a["rec"].ctypes.data_as(P(C.c_int64)), a["d2h"].ctypes.data_as(P(C.c_int64)),
                         a["h2d"].ctypes.data_as(P(C.c_int64)), a["bytes"].ctypes.data_as(P(C.c_uint64)),
                         a["in_ptr"].ctypes.data_as(P(C.c_int32)), a["in_idx"].ctypes.data_as(P(C.c_int32)),
                         a["need_ptr"].ctypes.data_as(P(C.c_int32)), a["need_idx"].ctypes.data_as(P(C.c_int32)),
                         int(resident), int(budget), int(tail), a["is_conv"].ctypes.data_as(P(C.c_uint8)),
                         0 if host_budget is None else int(host_budget), int(duplex[0]), int(duplex[1]))

    @staticmethod
    def from_dict(d, **kw):
        if "is_conv" in d and "is_conv" not in kw:
            kw["is_conv"] = d["is_conv"]
        return PlanProblem(d["fwd"], d["bwd"], d["bytes"], d["d2h"], d["h2d"], d["inputs"], d["needs"], **kw)

    def simulate(self, classes, sched=EAGER, events=False):
        n = self.n
        cls = np.asarray(classes, np.uint8)
        lo = np.zeros(n, np.uint8)
        li = np.zeros(n, np.uint8)
        stall = np.zeros(n, np.int64)
        cap = 8 * n + 16 if events else 0
        ev = {k: np.zeros(max(cap, 1), t) for k, t in
              (("lane", np.int32), ("kind", np.int32), ("id", np.int32), ("start", np.int64), ("end", np.int64))}
        r = SimResult()
        r.in_lo = lo.ctypes.data_as(P(C.c_uint8))
        r.in_li = li.ctypes.data_as(P(C.c_uint8))
        r.stall_ns = stall.ctypes.data_as(P(C.c_int64))
        r.events_cap = cap
        r.ev_lane = ev["lane"].ctypes.data_as(P(C.c_int32))
        r.ev_kind = ev["kind"].ctypes.data_as(P(C.c_int32))
        r.ev_id = ev["id"].ctypes.data_as(P(C.c_int32))
        r.ev_start = ev["start"].ctypes.data_as(P(C.c_int64))
        r.ev_end = ev["end"].ctypes.data_as(P(C.c_int64))
        check(lib.pooch_simulate(C.byref(self.c), cls.ctypes.data_as(P(C.c_uint8)), sched, C.byref(r)))
        out = {"oom": bool(r.oom), "makespan": int(r.makespan_ns), "peak": int(r.peak_bytes),
               "L_O": {int(i) for i in np.nonzero(lo)[0]}, "L_I": {int(i) for i in np.nonzero(li)[0]},
               "stall": {int(i): int(stall[i]) for i in range(n) if stall[i] >= 0 and cls[i] == SWAP}}
        if events:
            lanes = ("COMPUTE", "D2H", "H2D")
            k = min(r.n_events, cap)
            out["events"] = [(lanes[ev["lane"][i]], chr(ev["kind"][i]), int(ev["id"][i]), int(ev["start"][i]),
                              int(ev["end"][i])) for i in range(k)]
        return out

    def plan(self, strategy="pooch", li_cap=16, threads=0, sched=EAGER, fixed=None):
        n = self.n
        out = np.zeros(n, np.uint8)
        rep = PlanReport()
        cfg = SearchCfg(li_cap, threads, sched)
        fx = None if fixed is None else np.asarray(fixed, np.uint8)
        st = lib.pooch_plan_problem(C.byref(self.c), STRATEGIES[strategy], C.byref(cfg),
                                    None if fx is None else fx.ctypes.data_as(P(C.c_uint8)),
                                    out.ctypes.data_as(P(C.c_uint8)), C.byref(rep))
        if st == 2:
            return None, rep
        check(st)
        return [int(c) for c in out], rep

    def pack(self, classes, capacity, sched=EAGER):
        """Static offsets of every buffer instance (pooch_pack_problem); None if infeasible."""
        nb = 3 * self.n
        cls = np.asarray(classes, np.uint8)
        off = np.zeros(nb, np.uint64)
        a = np.zeros(nb, np.int32)
        f = np.zeros(nb, np.int32)
        sz = np.zeros(nb, np.uint64)
        hw = C.c_uint64()
        st = lib.pooch_pack_problem(C.byref(self.c), cls.ctypes.data_as(P(C.c_uint8)), sched, int(capacity),
                                    off.ctypes.data_as(P(C.c_uint64)), a.ctypes.data_as(P(C.c_int32)),
                                    f.ctypes.data_as(P(C.c_int32)), sz.ctypes.data_as(P(C.c_uint64)), C.byref(hw))
        if st == 2:
            return None
        check(st)
        return dict(offsets=off, alloc=a, free=f, sizes=sz, high_water=hw.value)

    def refine(self, classes, capacity, sched=EAGER):
        """The executor's plan refinement (pooch_refine_problem): (classes, makespan_ns, packs)."""
        cls = np.asarray(classes, np.uint8)
        out = np.zeros(self.n, np.uint8)
        mk = C.c_int64()
        pk = C.c_int32()
        check(lib.pooch_refine_problem(C.byref(self.c), cls.ctypes.data_as(P(C.c_uint8)), sched, int(capacity),
                                       out.ctypes.data_as(P(C.c_uint8)), C.byref(mk), C.byref(pk)))
        return [int(v) for v in out], int(mk.value), bool(pk.value)


def chrome_trace(events, names=None, pid=0, label=""):
    """Timeline events [(lane, kind, id, start_ns, end_ns)] -- pooch_simulate's (simulated) or
    pooch_last_trace's (measured) -- in the Chrome trace event format: complete events
    ("ph": "X") with ts / dur in microseconds, tid 0 = COMPUTE, 1 = D2H, 2 = H2D. Open the JSON in
    chrome://tracing or Perfetto; pass two timelines with different pids to overlay them."""
    tid = {"COMPUTE": 0, "D2H": 1, "H2D": 2}
    what = {"F": "fwd", "R": "recompute", "B": "bwd", "O": "swap-out", "I": "swap-in"}
    out = []
    for lane, kind, i, s, e in events:
        nm = names[i] if names is not None and 0 <= i < len(names) else str(i)
        out.append({"name": "%s %s" % (what.get(kind, kind), nm), "ph": "X", "ts": s / 1e3, "dur": max(e - s, 0) / 1e3,
                    "pid": pid, "tid": tid.get(lane, lane), "args": {"label": label}})
    return out
