// search.h — PAPER.md Algorithm 1 (heuristic search, §IV-B) over the selector's legal plans.
#pragma once
#include <cstdint>
#include <functional>
#include <vector>

#include "../../include/mbci.h"

namespace mbci {

struct SearchParams {
  int N = 512;           // population (SPEC.md default; the paper leaves it open)
  int n = 8;             // measured per round ("n is empirically set to 8")
  double eps = 0.01;     // relative convergence tolerance on the measured top-1
  uint64_t seed = 1;
  int max_rounds = 64;   // safety cap
  int model = 0;         // 0: the paper's t_estm (Eqs. 2-5); 1: the B200 score t_b200
};
struct SearchRound {
  double best_estimated = 0, top1_measured = 0, best_measured = 0;
  bool converged = false;
};
struct SearchLog {
  std::vector<SearchRound> rounds;
  int measurements = 0;
  double best_measured = 0;
  double history_min = 1e30;   // the historical minimum (Alg. 1 returns top1 on convergence)
};
using MeasureFn = std::function<double(const mbci_plan_t&)>;

// 0 on success (best_out set), -1 on bad arguments or an empty space.
int alg1_search(const std::vector<mbci_plan_t>& space, const SearchParams& sp, const MeasureFn& measure,
                mbci_plan_t* best_out, SearchLog* log);

}  // namespace mbci
