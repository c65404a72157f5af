// sim.cpp -- the simulator of sim.h. Rules (see oracle/sim.py for the reading of each):
//   program: F(0..n-1), then per backward task o (n-1..0) its missing recompute chain
//             and B(o);
//   deps:    swap-out after the last forward user; B/R after their swap-ins;
//   memory:  allocate at task start / swap-in issue, free at last use / swap-out end;
//   swap-in: FIFO in need order, eager = after the forward pass when the map fits together
//            with the compute program's look-ahead need, naive = when the task
//            before its first user starts.
#include <algorithm>
#include <climits>

#include "sim.h"

namespace pooch {

namespace {

struct Scratch {
  std::vector<ProgTask> prog;
  std::vector<uint8_t> regen;
  std::vector<int> consumers_max, last_fwd, need, last_bwd, bpos;
  std::vector<uint8_t> is_swap;
  std::vector<int64_t> A, Fr, S, V;
  std::vector<std::vector<int64_t>> sparse;
  std::vector<int> fifo;
  std::vector<std::vector<int>> ready_at, alloc_at, free_at;
  std::vector<int64_t> start_of, end_of, out_end, in_end, d_ready;
  std::vector<uint64_t> size;
};

thread_local Scratch tls;

void chain(const Problem& p, const uint8_t* cls, int m, Scratch& s) {
  for (int j : p.inputs[m])
    if (cls[j] == C_RECOMPUTE && !s.regen[j]) chain(p, cls, j, s);
  s.prog.push_back({'R', m});
  s.regen[m] = 1;
}

}  // namespace

void simulate(const Problem& p, const uint8_t* cls, const SimOptions& opt, SimOut& out) {
  Scratch& s = tls;
  const int n = p.n;
  out = SimOut();
  s.size.assign(n, 0);
  for (int m = 0; m < n; ++m) s.size[m] = cls[m] == C_FREE ? 0 : p.bytes[m];

  // ---- program
  s.prog.clear();
  s.regen.assign(n, 0);
  for (int i = 0; i < n; ++i) s.prog.push_back({'F', i});
  for (int o = n - 1; o >= 0; --o) {
    for (int m : p.needs[o])
      if (cls[m] == C_RECOMPUTE && !s.regen[m]) chain(p, cls, m, s);
    s.prog.push_back({'B', o});
  }
  const int P = (int)s.prog.size();

  // ---- uses
  s.consumers_max.assign(n, -1);
  s.last_fwd.resize(n);
  for (int c = 0; c < n; ++c)
    for (int m : p.inputs[c]) s.consumers_max[m] = std::max(s.consumers_max[m], c);
  for (int m = 0; m < n; ++m) s.last_fwd[m] = std::max(m, s.consumers_max[m]);
  s.need.assign(n, -1);
  s.last_bwd.assign(n, -1);
  s.bpos.assign(n, -1);
  for (int q = n; q < P; ++q) {
    const ProgTask& t = s.prog[q];
    const std::vector<int>& reads = t.kind == 'B' ? p.needs[t.id] : p.inputs[t.id];
    for (int m : reads) {
      if (s.need[m] < 0) s.need[m] = q;
      s.last_bwd[m] = q;
    }
    if (t.kind == 'B') s.bpos[t.id] = q;
  }
  s.is_swap.assign(n, 0);
  for (int m = 0; m < n; ++m) s.is_swap[m] = cls[m] == C_SWAP && s.need[m] >= 0;

  // ---- per-position allocation / compute-caused frees (and buffer lists for the ledger)
  s.A.assign(P, 0);
  s.Fr.assign(P, 0);
  const bool L = opt.record_ledger;
  if (L) {
    s.alloc_at.assign(P, {});
    s.free_at.assign(P, {});
  }
  for (int q = 0; q < P; ++q) {
    const ProgTask& t = s.prog[q];
    if (t.kind == 'F') {
      s.A[q] += s.size[t.id];
      if (L) s.alloc_at[q].push_back(t.id);
    } else if (t.kind == 'R') {
      s.A[q] += s.size[t.id];
      if (L) s.alloc_at[q].push_back(n + t.id);
    }
  }
  for (int m = 0; m < n; ++m) {
    if (s.consumers_max[m] >= 0) {
      int a = s.bpos[s.consumers_max[m]], f = s.bpos[m];
      s.A[a] += p.bytes[m];
      s.Fr[f] += p.bytes[m];
      if (L) {
        s.alloc_at[a].push_back(2 * n + m);
        s.free_at[f].push_back(2 * n + m);
      }
    }
  }
  for (int m = 0; m < n; ++m) {
    uint8_t c = cls[m];
    if (s.need[m] < 0) {
      s.Fr[s.last_fwd[m]] += s.size[m];
      if (L) s.free_at[s.last_fwd[m]].push_back(m);
    } else if (c == C_KEEP || c == C_FREE) {
      s.Fr[s.last_bwd[m]] += s.size[m];
      if (L) s.free_at[s.last_bwd[m]].push_back(m);
    } else if (c == C_SWAP) {
      s.Fr[s.last_bwd[m]] += s.size[m];
      if (L) s.free_at[s.last_bwd[m]].push_back(n + m);
    } else {
      s.Fr[s.last_fwd[m]] += s.size[m];
      s.Fr[s.last_bwd[m]] += s.size[m];
      if (L) {
        s.free_at[s.last_fwd[m]].push_back(m);
        s.free_at[s.last_bwd[m]].push_back(n + m);
      }
    }
  }
  // look-ahead table: V[q] = S[q] + A[q], S[q] = sum_{j<q} (A[j] - Fr[j]); sparse table for max
  s.S.assign(P + 1, 0);
  for (int q = 0; q < P; ++q) s.S[q + 1] = s.S[q] + s.A[q] - s.Fr[q];
  int LOG = 1;
  while ((1 << LOG) <= P) ++LOG;
  if ((int)s.sparse.size() < LOG) s.sparse.resize(LOG);
  s.sparse[0].resize(P);
  for (int q = 0; q < P; ++q) s.sparse[0][q] = s.S[q] + s.A[q];
  for (int k = 1; k < LOG; ++k) {
    s.sparse[k].resize(P);
    for (int q = 0; q + (1 << k) <= P; ++q)
      s.sparse[k][q] = std::max(s.sparse[k - 1][q], s.sparse[k - 1][q + (1 << (k - 1))]);
  }
  auto range_max = [&](int a, int b) {  // inclusive
    int k = 31 - __builtin_clz((unsigned)(b - a + 1));
    return std::max(s.sparse[k][a], s.sparse[k][b - (1 << k) + 1]);
  };

  auto dur = [&](const ProgTask& t) -> int64_t {
    return t.kind == 'F' ? p.fwd[t.id] : (t.kind == 'R' ? p.rec[t.id] : p.bwd[t.id]);
  };

  s.fifo.clear();
  for (int m = 0; m < n; ++m)
    if (s.is_swap[m]) s.fifo.push_back(m);
  std::sort(s.fifo.begin(), s.fifo.end(), [&](int a, int b) {
    return s.need[a] != s.need[b] ? s.need[a] < s.need[b] : a < b;
  });
  if (p.host_budget > 0) {  // the swap class must fit the pinned host arena (Reading 36)
    uint64_t hb = 0;
    for (int m : s.fifo) hb += p.bytes[m];
    if (hb > p.host_budget) {
      out.oom = true;
      return;
    }
  }
  s.ready_at.assign(n, {});
  for (int m = 0; m < n; ++m)
    if (s.is_swap[m]) s.ready_at[s.last_fwd[m]].push_back(m);

  // ---- event loop
  const uint64_t budget = p.budget;
  int64_t t = 0;
  uint64_t live = p.resident, peak = live;
  int pc = 0;
  int c_q = -1;
  int64_t c_end = 0;
  s.start_of.assign(P, -1);
  s.end_of.assign(P, -1);
  // copy lanes: remaining work in ns x 1000 and the start event's index (its end is set at
  // completion); while both lanes are busy each progresses at its duplex rate (Reading 51)
  int d_m = -1;
  int64_t d_rem = 0;
  size_t d_ev = 0;
  s.d_ready.assign(n, -1);
  int n_ready = 0;
  s.out_end.assign(n, -1);
  int h_m = -1;
  int64_t h_rem = 0;
  size_t h_ev = 0;
  const int64_t dx_d = p.duplex_d2h > 0 ? p.duplex_d2h : 1000, dx_h = p.duplex_h2d > 0 ? p.duplex_h2d : 1000;
  size_t hq = 0;
  s.in_end.assign(n, -1);
  int fwd_done = 0;
  int64_t fwd_end = -1;
  std::vector<SimEvent>& ev = out.events;
  std::vector<LedgerEntry>& led = out.ledger;
  const bool E = opt.record_events;

  while (true) {
    // completions at t: COMPUTE, D2H, H2D
    if (c_q >= 0 && c_end == t) {
      int q = c_q;
      s.end_of[q] = t;
      live -= s.Fr[q];
      if (L)
        for (int b : s.free_at[q]) led.push_back({t, b, false, 0, 0, s.prog[q].kind, s.prog[q].id});
      c_q = -1;
      if (s.prog[q].kind == 'F') {
        ++fwd_done;
        for (int m : s.ready_at[q]) {
          s.d_ready[m] = t;
          ++n_ready;
        }
        if (fwd_done == n) fwd_end = t;
      }
    }
    if (d_m >= 0 && d_rem <= 0) {
      live -= s.size[d_m];
      s.out_end[d_m] = t;
      if (E) ev[d_ev].end = t;
      if (L) led.push_back({t, d_m, false, 0, 1, 'O', d_m});
      d_m = -1;
    }
    if (h_m >= 0 && h_rem <= 0) {
      s.in_end[h_m] = t;
      if (E) ev[h_ev].end = t;
      h_m = -1;
    }
    // starts at t: COMPUTE, D2H, H2D
    if (c_q < 0 && pc < P) {
      const ProgTask& tk = s.prog[pc];
      bool ok = true;
      if (tk.kind != 'F') {
        const std::vector<int>& reads = tk.kind == 'B' ? p.needs[tk.id] : p.inputs[tk.id];
        for (int m : reads)
          if (s.is_swap[m] && (s.in_end[m] < 0 || s.in_end[m] > t)) ok = false;
      }
      if (ok && live + (uint64_t)s.A[pc] <= budget) {
        live += s.A[pc];
        peak = std::max(peak, live);
        s.start_of[pc] = t;
        c_q = pc;
        c_end = t + dur(tk);
        if (E) ev.push_back({0, tk.kind, tk.id, t, c_end});
        if (L)
          for (int b : s.alloc_at[pc]) led.push_back({t, b, true, 0, 0, tk.kind, tk.id});
        ++pc;
      }
    }
    if (d_m < 0 && n_ready > 0) {
      int best = -1;
      for (int m = 0; m < n; ++m)
        if (s.d_ready[m] >= 0 && (best < 0 || s.d_ready[m] < s.d_ready[best])) best = m;
      d_m = best;
      s.d_ready[best] = -1;
      --n_ready;
      d_rem = 1000 * p.d2h[best];
      d_ev = ev.size();
      if (E) ev.push_back({1, 'O', best, t, -1});
    }
    if (h_m < 0 && hq < s.fifo.size()) {
      int m = s.fifo[hq];
      bool phase_ok;
      if (opt.sched == SCHED_EAGER) {
        phase_ok = fwd_end >= 0 && fwd_end <= t;
      } else {
        int trig = s.need[m] - 1;
        if (opt.sched == SCHED_SN) {  // the preceding convolution's backward task
          trig = n - 1;
          for (int q = s.need[m] - 1; q >= n; --q)
            if (s.prog[q].kind == 'B' && !p.is_conv.empty() && p.is_conv[s.prog[q].id]) {
              trig = q;
              break;
            }
        }
        phase_ok = s.start_of[trig] >= 0 && s.start_of[trig] <= t;
      }
      if (phase_ok && s.out_end[m] >= 0 && s.out_end[m] <= t) {
        int64_t head = std::max<int64_t>(0, range_max(pc, s.need[m]) - s.S[pc]);
        if (live + s.size[m] + (uint64_t)head <= budget) {
          live += s.size[m];
          peak = std::max(peak, live);
          h_m = m;
          h_rem = 1000 * p.h2d[m];
          h_ev = ev.size();
          if (E) ev.push_back({2, 'I', m, t, -1});
          if (L) led.push_back({t, n + m, true, 0, 2, 'I', m});
          ++hq;
        }
      }
    }
    // advance
    const bool both = d_m >= 0 && h_m >= 0;
    const int64_t rd = both ? dx_d : 1000, rh = both ? dx_h : 1000;
    int64_t nxt = INT64_MAX;
    if (c_q >= 0) nxt = std::min(nxt, c_end);
    if (d_m >= 0) nxt = std::min(nxt, t + (d_rem + rd - 1) / rd);
    if (h_m >= 0) nxt = std::min(nxt, t + (h_rem + rh - 1) / rh);
    if (nxt == INT64_MAX) {
      if (pc < P || hq < s.fifo.size() || n_ready > 0) out.oom = true;
      break;
    }
    if (d_m >= 0) d_rem -= (nxt - t) * rd;
    if (h_m >= 0) h_rem -= (nxt - t) * rh;
    t = nxt;
  }

  out.peak = peak;
  if (E) out.program = s.prog;
  if (out.oom) return;
  out.makespan = t;  // the loop ends at the last completion
  out.fwd_end = fwd_end;
  if (L)
    for (LedgerEntry& e : led) {
      int b = e.buf;
      e.bytes = b < n ? s.size[b] : (b < 2 * n ? s.size[b - n] : p.bytes[b - 2 * n]);
    }
  if (opt.want_sets) {
    out.stall.assign(n, -1);
    out.lo.assign(n, 0);
    out.li.assign(n, 0);
    for (int m : s.fifo) {
      int q = s.need[m];
      int64_t lane_ready = s.end_of[q - 1];
      out.stall[m] = std::max<int64_t>(0, s.in_end[m] - lane_ready);
      if (out.stall[m] > 0) out.li[m] = 1;
      if (s.out_end[m] > fwd_end) out.lo[m] = 1;
    }
  }
}

int64_t sim_makespan(const Problem& p, const std::vector<uint8_t>& cls, int sched) {
  SimOptions o;
  o.sched = sched;
  o.want_sets = false;
  SimOut r;
  simulate(p, cls.data(), o, r);
  return r.oom ? -1 : r.makespan;
}

}  // namespace pooch
