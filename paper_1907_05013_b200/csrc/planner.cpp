// planner.cpp -- PoocH classification (Sec. 4.4) over the simulator, plus the
// comparison strategies of Sec. 5.1 and an exhaustive search for tiny nets.
// Must return exactly the class vector of oracle/planner.py on every profile.
//
// Step 1 (Sec. 4.4.2): simulate all-swap; maps outside L_O u L_I stay swap;
//   enumerate the binary tree over L_I (capped at li_cap by stall rank); at every leaf
//   scan L_O \ L_I from the output layer flipping swap -> keep, reverting
//   flips that run out of memory; keep the recorded state with minimal makespan.
// Step 2 (Sec. 4.4.3, Eq. (1)): r(X) = recompute_overhead / swap_overhead, both
//   against the makespan with X free of cost; drop r >= 1, commit argmin r < 1; repeat.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <thread>

#include "common.h"
#include "planner.h"

namespace pooch {

namespace {

struct Key {
  int64_t ms;
  int keeps;
  std::vector<uint8_t> cls;
  bool operator<(const Key& o) const {
    if (ms != o.ms) return ms < o.ms;
    if (keeps != o.keeps) return keeps < o.keeps;
    return cls < o.cls;
  }
};

int count_keep(const std::vector<uint8_t>& c) { return (int)std::count(c.begin(), c.end(), (uint8_t)C_KEEP); }

int hw_threads(int want) {
  if (want > 0) return want;
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)std::min(h, 64u) : 4;
}

template <class F>
void parallel_for(int n, int threads, F&& f) {
  threads = std::max(1, std::min(threads, n));
  if (threads == 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int> next(0);
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t)
    ts.emplace_back([&] {
      for (int i; (i = next.fetch_add(1)) < n;) f(i);
    });
  for (auto& t : ts) t.join();
}

}  // namespace

int64_t Planner::ms(const std::vector<uint8_t>& cls) {
  ++sims_;
  return sim_makespan(p_, cls, sched_);
}

// Step 1's starting point: all-swap, or -- when its swap class exceeds the pinned
// host arena (Reading 37) -- all-swap with the cheapest-to-replay maps (recompute ns per byte;
// ties: larger bytes, smaller id; never the sink) moved to recompute until it fits, the sink
// kept if it alone does not fit.
static std::vector<uint8_t> host_fit_base(const Problem& p) {
  const int n = p.n;
  std::vector<uint8_t> cls(n, C_SWAP);
  if (p.host_budget == 0) return cls;
  uint64_t total = 0;
  for (int m = 0; m < n; ++m) total += p.bytes[m];
  std::vector<int> order;
  for (int m = 0; m + 1 < n; ++m) order.push_back(m);
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    double ra = (double)p.rec[a] / (double)std::max<uint64_t>(p.bytes[a], 1);
    double rb = (double)p.rec[b] / (double)std::max<uint64_t>(p.bytes[b], 1);
    if (ra != rb) return ra < rb;
    if (p.bytes[a] != p.bytes[b]) return p.bytes[a] > p.bytes[b];
    return a < b;
  });
  for (int m : order) {
    if (total <= p.host_budget) break;
    cls[m] = C_RECOMPUTE;
    total -= p.bytes[m];
  }
  // the sink is never recompute; if it alone still exceeds the host arena (e.g. none at all) it
  // is kept, so a context without a pinned host arena still gets keep / recompute plans
  if (total > p.host_budget) cls[n - 1] = C_KEEP;
  return cls;
}

bool Planner::step1(std::vector<uint8_t>& best_cls, int64_t& best_ms) {
  const int n = p_.n;
  std::vector<uint8_t> all_swap = host_fit_base(p_);
  SimOptions o;
  o.sched = sched_;
  SimOut base;
  simulate(p_, all_swap.data(), o, base);
  sims_++;
  if (base.oom) return false;
  std::vector<int> LI, LO;
  for (int m = 0; m < n; ++m) {
    if (base.li[m]) LI.push_back(m);
    if (base.lo[m]) LO.push_back(m);
  }
  lo_size_ = (int)LO.size();
  li_size_ = (int)LI.size();
  std::vector<int> ranked = LI;
  std::sort(ranked.begin(), ranked.end(), [&](int a, int b) {
    return base.stall[a] != base.stall[b] ? base.stall[a] > base.stall[b] : a < b;
  });
  int cap = std::max(0, cfg_.li_cap);
  std::vector<int> tree(ranked.begin(), ranked.begin() + std::min<int>(cap, (int)ranked.size()));
  std::sort(tree.begin(), tree.end());
  std::vector<uint8_t> in_tree(n, 0), in_scan(n, 0);
  for (int m : tree) in_tree[m] = 1;
  for (size_t i = tree.size(); i < ranked.size(); ++i) in_scan[ranked[i]] = 1;
  for (int m : LO)
    if (!in_tree[m]) in_scan[m] = 1;
  std::vector<int> scan;
  for (int m = n - 1; m >= 0; --m)
    if (in_scan[m]) scan.push_back(m);

  const int64_t leaves = int64_t(1) << tree.size();  // tree.size() <= li_cap <= kMaxLiCap
  const int T = hw_threads(cfg_.threads);
  std::vector<Key> best_per_thread;
  // deterministic reduction: each leaf's best, reduced in leaf order via min (total order)
  std::vector<Key> leaf_best((size_t)leaves);
  std::vector<int64_t> leaf_sims((size_t)leaves, 0);
  parallel_for((int)leaves, T, [&](int leaf) {
    std::vector<uint8_t> cls = all_swap;
    for (size_t b = 0; b < tree.size(); ++b)
      if ((leaf >> b) & 1) cls[tree[b]] = C_KEEP;
    Key kb{INT64_MAX, INT_MAX, {}};
    int64_t m0 = sim_makespan(p_, cls, sched_);
    int64_t s = 1;
    if (m0 >= 0) kb = Key{m0, count_keep(cls), cls};
    for (int m : scan) {
      cls[m] = C_KEEP;
      int64_t m2 = sim_makespan(p_, cls, sched_);
      ++s;
      if (m2 < 0) {
        cls[m] = C_SWAP;
        continue;
      }
      Key k{m2, count_keep(cls), cls};
      if (k < kb) kb = k;
    }
    leaf_best[leaf] = std::move(kb);
    leaf_sims[leaf] = s;
  });
  Key best{base.makespan, 0, all_swap};
  for (int64_t l = 0; l < leaves; ++l) {
    sims_ += leaf_sims[l];
    if (leaf_best[l].ms != INT64_MAX && leaf_best[l] < best) best = leaf_best[l];
  }
  best_cls = best.cls;
  best_ms = best.ms;
  return true;
}

void Planner::step2(std::vector<uint8_t>& cls, int64_t& t_swap) {
  const int n = p_.n;
  std::vector<int> L;
  for (int m = 0; m < n - 1; ++m)
    if (cls[m] == C_SWAP) L.push_back(m);
  t_swap = ms(cls);
  const int T = hw_threads(cfg_.threads);
  while (!L.empty()) {
    std::vector<double> r(L.size());
    std::vector<int64_t> trec(L.size());
    parallel_for((int)L.size(), T, [&](int i) {
      int X = L[i];
      std::vector<uint8_t> c0 = cls, cr = cls;
      c0[X] = C_FREE;
      cr[X] = C_RECOMPUTE;
      int64_t t0 = sim_makespan(p_, c0, sched_);
      int64_t tr = sim_makespan(p_, cr, sched_);
      int64_t swap_ov = t0 < 0 ? 0 : std::max<int64_t>(0, t_swap - t0);
      double rec_ov = tr < 0 ? INFINITY : (double)std::max<int64_t>(0, tr - t0);
      r[i] = swap_ov == 0 ? INFINITY : rec_ov / (double)swap_ov;
      trec[i] = tr;
    });
    sims_ += 2 * (int64_t)L.size();
    std::vector<int> keep_going;
    int pick = -1;
    for (size_t i = 0; i < L.size(); ++i) {
      if (!(r[i] < 1.0)) continue;
      keep_going.push_back((int)i);
      if (pick < 0) {
        pick = (int)i;
        continue;
      }
      int a = L[i], b = L[pick];
      if (r[i] < r[pick] || (r[i] == r[pick] && (p_.bytes[a] > p_.bytes[b] || (p_.bytes[a] == p_.bytes[b] && a < b))))
        pick = (int)i;
    }
    if (pick < 0) break;
    int X = L[pick];
    cls[X] = C_RECOMPUTE;
    t_swap = trec[pick];
    decisions_.push_back({X, r[pick]});
    std::vector<int> nl;
    for (int i : keep_going)
      if (L[i] != X) nl.push_back(L[i]);
    L.swap(nl);
  }
}

pooch_status Planner::run(int strategy, const uint8_t* fixed, std::vector<uint8_t>& cls, int64_t& makespan) {
  const int n = p_.n;
  auto t0 = std::chrono::steady_clock::now();
  sims_ = 0;
  pooch_status st = POOCH_OK;
  makespan = -1;
  switch (strategy) {
    case POOCH_STRAT_INCORE:
      cls.assign(n, C_KEEP);
      makespan = ms(cls);
      break;
    case POOCH_STRAT_SWAP_ALL_NAIVE:
      cls.assign(n, C_SWAP);
      sched_ = SCHED_NAIVE;
      makespan = ms(cls);
      break;
    case POOCH_STRAT_SWAP_ALL:
      cls.assign(n, C_SWAP);
      makespan = ms(cls);
      break;
    case POOCH_STRAT_FIXED:
      if (!fixed) return fail(POOCH_EUSAGE, "STRAT_FIXED needs fixed_classes");
      cls.assign(fixed, fixed + n);
      for (uint8_t c : cls)
        if (c > C_RECOMPUTE) return fail(POOCH_EUSAGE, "class value out of range");
      if (cls[n - 1] == C_RECOMPUTE) return fail(POOCH_EUSAGE, "the sink map cannot be recompute");
      makespan = ms(cls);
      break;
    case POOCH_STRAT_SWAP_OPT:
    case POOCH_STRAT_POOCH: {
      cls.assign(n, C_KEEP);
      int64_t mk = ms(cls);
      if (mk >= 0) {  // in-core fits: nothing to classify
        makespan = mk;
        break;
      }
      int64_t m1;
      if (!step1(cls, m1)) {
        cls.clear();
        break;
      }
      makespan = m1;
      if (strategy == POOCH_STRAT_POOCH) step2(cls, makespan);
      break;
    }
    case POOCH_STRAT_EXHAUSTIVE: {
      if (n > 12) return fail(POOCH_EUSAGE, "exhaustive search is limited to n <= 12 (n = %d)", n);
      int64_t total = 2;
      for (int i = 0; i < n - 1; ++i) total *= 3;
      const int T = hw_threads(cfg_.threads);
      std::vector<Key> best_t(T, Key{INT64_MAX, INT_MAX, {}});
      std::atomic<int64_t> next(0);
      std::vector<std::thread> ts;
      for (int t = 0; t < T; ++t)
        ts.emplace_back([&, t] {
          std::vector<uint8_t> c(n);
          for (int64_t i; (i = next.fetch_add(1)) < total;) {
            int64_t v = i;
            c[n - 1] = (uint8_t)(v % 2);  // sink: keep / swap
            v /= 2;
            for (int k = n - 2; k >= 0; --k) {
              c[k] = (uint8_t)(v % 3);
              v /= 3;
            }
            int64_t m = sim_makespan(p_, c, sched_);
            if (m < 0) continue;
            Key k{m, count_keep(c), c};
            if (k < best_t[t]) best_t[t] = k;
          }
        });
      for (auto& t : ts) t.join();
      sims_ += total;
      Key best{INT64_MAX, INT_MAX, {}};
      for (auto& k : best_t)
        if (k.ms != INT64_MAX && k < best) best = k;
      if (best.ms != INT64_MAX) {
        cls = best.cls;
        makespan = best.ms;
      } else {
        cls.clear();
      }
      break;
    }
    case POOCH_STRAT_SUPERNEURONS: {
      // keep from the output layer while resident + kept bytes fit;
      // the rest: convolution outputs swap, others recompute; swap-in with the preceding conv.
      cls.assign(n, 255);
      uint64_t kept = p_.resident;
      for (int m = n - 1; m >= 0; --m) {
        if (kept + p_.bytes[m] > p_.budget) break;
        cls[m] = C_KEEP;
        kept += p_.bytes[m];
      }
      for (int m = 0; m < n; ++m)
        if (cls[m] == 255) cls[m] = ((!p_.is_conv.empty() && p_.is_conv[m]) || m == n - 1) ? C_SWAP : C_RECOMPUTE;
      sched_ = SCHED_SN;
      makespan = ms(cls);
      break;
    }
    default:
      return fail(POOCH_EUSAGE, "unknown strategy %d", strategy);
  }
  wall_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (cls.empty() || makespan < 0) st = fail(POOCH_EINFEASIBLE, "no classification fits the budget");
  return st;
}

void Planner::report(const std::vector<uint8_t>& cls, int64_t makespan, pooch_plan_report* r) const {
  if (!r) return;
  *r = pooch_plan_report{};
  r->feasible = !cls.empty() && makespan >= 0;
  r->n_sims = sims_;
  r->wall_ms = wall_ms_;
  r->lo_size = lo_size_;
  r->li_size = li_size_;
  if (!r->feasible) return;
  r->makespan_ns = makespan + p_.tail;
  SimOptions o;
  o.sched = sched_;
  o.want_sets = false;
  SimOut s;
  simulate(p_, cls.data(), o, s);
  r->peak_bytes = s.peak;
  for (size_t m = 0; m < cls.size(); ++m) {
    if (cls[m] == C_KEEP) r->n_keep++;
    if (cls[m] == C_SWAP) {
      r->n_swap++;
      r->host_bytes += p_.bytes[m];
    }
    if (cls[m] == C_RECOMPUTE) r->n_recompute++;
  }
}

}  // namespace pooch

using namespace pooch;

extern "C" pooch_status pooch_simulate(const pooch_problem* prob, const uint8_t* classes, int32_t sched,
                                       pooch_sim_result* out) {
  if (!prob || !classes || !out) return fail(POOCH_EUSAGE, "null argument");
  Problem p;
  std::string err;
  if (!problem_from_c(*prob, p, err)) return fail(POOCH_EUSAGE, "%s", err.c_str());
  for (int i = 0; i < p.n; ++i)
    if (classes[i] > C_FREE) return fail(POOCH_EUSAGE, "class value out of range");
  SimOptions o;
  o.sched = sched == POOCH_SCHED_NAIVE ? SCHED_NAIVE : (sched == POOCH_SCHED_SN ? SCHED_SN : SCHED_EAGER);
  o.record_events = out->events_cap > 0;
  SimOut s;
  simulate(p, classes, o, s);
  out->oom = s.oom ? 1 : 0;
  out->makespan_ns = s.makespan;
  out->peak_bytes = s.peak;
  out->n_events = (int32_t)s.events.size();
  if (!s.oom) {
    for (int m = 0; m < p.n; ++m) {
      if (out->in_lo) out->in_lo[m] = s.lo[m];
      if (out->in_li) out->in_li[m] = s.li[m];
      if (out->stall_ns) out->stall_ns[m] = s.stall[m];
    }
  }
  int k = 0;
  for (const SimEvent& e : s.events) {
    if (k >= out->events_cap) break;
    if (out->ev_lane) out->ev_lane[k] = e.lane;
    if (out->ev_kind) out->ev_kind[k] = e.kind;
    if (out->ev_id) out->ev_id[k] = e.id;
    if (out->ev_start) out->ev_start[k] = e.start;
    if (out->ev_end) out->ev_end[k] = e.end;
    ++k;
  }
  return POOCH_OK;
}

extern "C" pooch_status pooch_plan_problem(const pooch_problem* prob, int32_t strategy, const pooch_search_cfg* cfg,
                                           const uint8_t* fixed_classes, uint8_t* classes_out,
                                           pooch_plan_report* report) {
  if (!prob) return fail(POOCH_EUSAGE, "null problem");
  Problem p;
  std::string err;
  if (!problem_from_c(*prob, p, err)) return fail(POOCH_EUSAGE, "%s", err.c_str());
  pooch_search_cfg c = cfg ? *cfg : pooch_search_cfg{16, 0, POOCH_SCHED_EAGER};
  if (c.li_cap < 0 || c.li_cap > kMaxLiCap) return fail(POOCH_EUSAGE, "li_cap must be in [0, %d]", kMaxLiCap);
  Planner pl(p, c);
  std::vector<uint8_t> cls;
  int64_t mk;
  pooch_status st = pl.run(strategy, fixed_classes, cls, mk);
  pl.report(cls, mk, report);
  if (st == POOCH_OK && classes_out) std::copy(cls.begin(), cls.end(), classes_out);
  return st;
}
