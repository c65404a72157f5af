// sim.h -- discrete-event timeline + memory simulator of one iteration (Sec. 4.1.2;
// swap-in scheduling Sec. 4.3). Semantics are specified in oracle/sim.py's docstring and
// DESIGN.md "Simulator"; this implementation must agree with it exactly (tolerance 0).
#pragma once
#include <cstdint>
#include <vector>

#include "graph.h"

namespace pooch {

enum : uint8_t { C_KEEP = 0, C_SWAP = 1, C_RECOMPUTE = 2, C_FREE = 3 };
enum : int { SCHED_EAGER = 0, SCHED_NAIVE = 1, SCHED_SN = 2 };

struct SimEvent {
  int lane;   // 0 COMPUTE, 1 D2H, 2 H2D
  char kind;  // 'F','B','R','O','I'
  int id;
  int64_t start, end;
};

// Buffer instances: fwd instance of map m = m, backward-phase instance (swap-in or
// recompute) = n + m, gradient of map m = 2n + m.
struct LedgerEntry {
  int64_t t;
  int buf;
  bool alloc;
  uint64_t bytes;
  int lane;   // op performing the alloc / free: lane, kind, id
  char kind;
  int id;
};

struct ProgTask {
  char kind;  // 'F', 'R', 'B'
  int id;
};

struct SimOut {
  bool oom = false;
  int64_t makespan = 0;
  uint64_t peak = 0;
  int64_t fwd_end = 0;
  std::vector<int64_t> stall;   // per map, -1 if not swapped in
  std::vector<uint8_t> lo, li;  // membership of L_O / L_I
  std::vector<SimEvent> events; // when record_events
  std::vector<LedgerEntry> ledger;  // when record_ledger
  std::vector<ProgTask> program;    // when record_events
};

struct SimOptions {
  int sched = SCHED_EAGER;
  bool record_events = false;
  bool record_ledger = false;
  bool want_sets = true;
};

void simulate(const Problem& p, const uint8_t* cls, const SimOptions& opt, SimOut& out);

// Convenience: makespan or -1 on OOM.
int64_t sim_makespan(const Problem& p, const std::vector<uint8_t>& cls, int sched = SCHED_EAGER);

}  // namespace pooch
