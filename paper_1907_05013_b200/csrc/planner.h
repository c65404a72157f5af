// planner.h -- keep / swap / recompute classification (Sec. 4.4).
#pragma once
#include <vector>

#include "../../include/pooch.h"
#include "sim.h"

namespace pooch {

// Largest accepted L_I tree cap (Reading 16): 2^20 leaves, each a scan of simulations.
constexpr int kMaxLiCap = 20;

struct Decision {
  int map;
  double r;  // Eq. (1) ratio at commit time
};

class Planner {
 public:
  Planner(const Problem& p, const pooch_search_cfg& cfg)
      : p_(p),
        cfg_(cfg),
        sched_(cfg.sched == POOCH_SCHED_NAIVE ? SCHED_NAIVE : (cfg.sched == POOCH_SCHED_SN ? SCHED_SN : SCHED_EAGER)) {}
  // Fills cls (empty when infeasible) and the simulated makespan (without tail).
  pooch_status run(int strategy, const uint8_t* fixed, std::vector<uint8_t>& cls, int64_t& makespan);
  void report(const std::vector<uint8_t>& cls, int64_t makespan, pooch_plan_report* r) const;
  int sched() const { return sched_; }
  const std::vector<Decision>& decisions() const { return decisions_; }

 private:
  int64_t ms(const std::vector<uint8_t>& cls);
  bool step1(std::vector<uint8_t>& cls, int64_t& makespan);
  void step2(std::vector<uint8_t>& cls, int64_t& makespan);

  const Problem& p_;
  pooch_search_cfg cfg_;
  int sched_;
  int64_t sims_ = 0;
  double wall_ms_ = 0;
  int lo_size_ = 0, li_size_ = 0;
  std::vector<Decision> decisions_;
};

}  // namespace pooch
