// search.cpp — PAPER.md Algorithm 1 (§IV-B): population-based heuristic search that
// ranks candidates with the analytical model and measures only the top n of each round.
//
//   population = generateCandidates(P, N)                         (line 1: N random candidates)
//   loop: estimate all, sort ascending, measure the top n          (lines 5-8)
//         if difference(top1_t, best_t) < eps: best = top1, stop  (lines 10-12; relative difference,
//                                                                   SPEC.md reading)
//         if top1_t < best_t: best = top1                          (lines 13-16)
//         population = mutate(population, weight = 1 / et)         (line 17: N weighted draws, each
//                                                                   mutates ONE tile parameter to an
//                                                                   adjacent legal value)
// The search space is the pruned, legal plan list of enumerate_plans (Rules 1-4); the
// tile "loops" a mutation may move are BN (the n tile), TL (the h tile) and the pipeline depth;
// the kernel family plays the role of the tiling expression and is never mutated.
// Measurement is a caller-supplied callback (GPU timing in mbci_chain_create with tune = 2, or a
// synthetic function in the CPU tests); measured plans are cached, so a plan is timed once.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <tuple>
#include <vector>

#include "search.h"

namespace mbci {

namespace {

// splitmix64: one seeded stream, consumed only at the round barrier (deterministic per seed)
struct Rng {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
  int below(int n) { return static_cast<int>(next() % static_cast<uint64_t>(n)); }
};

using Key = std::tuple<int32_t, int32_t, int32_t, int32_t>;   // kernel, BN, TL, stages
Key key_of(const mbci_plan_t& p) { return Key{p.kernel, p.BN, p.TL, p.stages}; }

double estimate(const mbci_plan_t& p, int model) { return model == 0 ? p.t_estm : p.t_b200; }

}  // namespace

int alg1_search(const std::vector<mbci_plan_t>& space, const SearchParams& sp, const MeasureFn& measure,
                mbci_plan_t* best_out, SearchLog* log) {
  if (space.empty() || sp.N < 1 || sp.n < 1 || !(sp.eps > 0.0) || sp.max_rounds < 1) return -1;
  std::map<Key, int> index;
  for (int i = 0; i < static_cast<int>(space.size()); ++i) index.emplace(key_of(space[i]), i);
  // adjacent legal values of the three tile parameters (ladders over the legal space)
  Rng rng{sp.seed};
  std::vector<int> pop;
  // line 1: N random candidates (the whole space when it is smaller than N)
  if (static_cast<int>(space.size()) <= sp.N) {
    for (int i = 0; i < static_cast<int>(space.size()); ++i) pop.push_back(i);
  } else {
    for (int k = 0; k < sp.N; ++k) pop.push_back(rng.below(static_cast<int>(space.size())));
  }
  std::map<int, double> measured;   // plan index -> seconds (cache)
  double best_t = 1e9;              // line 2
  int best = -1;                    // line 3
  if (log) *log = SearchLog{};
  for (int round = 0; round < sp.max_rounds; ++round) {
    // lines 5-7: estimate, sort ascending, take the n best-estimated distinct candidates
    std::vector<int> order(pop);
    std::sort(order.begin(), order.end());
    order.erase(std::unique(order.begin(), order.end()), order.end());
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return estimate(space[a], sp.model) < estimate(space[b], sp.model);
    });
    const int k = std::min<int>(sp.n, static_cast<int>(order.size()));
    // line 8: measure
    double top1_t = 1e30;
    int top1 = -1;
    for (int i = 0; i < k; ++i) {
      const int c = order[i];
      auto it = measured.find(c);
      double t;
      if (it != measured.end()) {
        t = it->second;
      } else {
        t = measure(space[c]);
        measured.emplace(c, t);
        if (log) ++log->measurements;
      }
      if (t < top1_t) {
        top1_t = t;
        top1 = c;
      }
    }
    if (top1 < 0) return -1;
    const bool converged = best >= 0 && std::fabs(top1_t - best_t) / best_t < sp.eps;   // line 10
    if (log) {
      SearchRound r;
      r.best_estimated = estimate(space[order[0]], sp.model);
      r.top1_measured = top1_t;
      r.best_measured = std::min(best_t, top1_t);
      r.converged = converged;
      log->rounds.push_back(r);
      log->history_min = std::min(log->history_min, top1_t);
    }
    if (converged) {   // lines 11-12: the paper returns top1 on convergence
      best = top1;
      best_t = top1_t;
      break;
    }
    if (top1_t < best_t) {   // lines 13-16
      best = top1;
      best_t = top1_t;
    }
    // line 17: N draws weighted by 1 / et, each mutating one tile parameter to an adjacent legal
    // value (bounded retries; the parent passes through when none is legal)
    std::vector<double> cum;
    double acc = 0.0;
    for (int c : pop) {
      acc += 1.0 / std::max(estimate(space[c], sp.model), 1e-15);
      cum.push_back(acc);
    }
    std::vector<int> next;
    for (int d = 0; d < sp.N; ++d) {
      const double u = rng.uniform() * acc;
      const int parent = pop[std::lower_bound(cum.begin(), cum.end(), u) - cum.begin()];
      const mbci_plan_t& pp = space[parent];
      int child = parent;
      for (int attempt = 0; attempt < 8 && child == parent; ++attempt) {
        Key kk = key_of(pp);
        const int axis = rng.below(3), dir = (rng.next() & 1) ? 1 : -1;
        if (axis == 0) std::get<1>(kk) = dir > 0 ? std::get<1>(kk) * 2 : std::get<1>(kk) / 2;   // BN ladder x2
        else if (axis == 1) std::get<2>(kk) += 16 * dir;                                       // TL ladder 16
        else std::get<3>(kk) += dir;                                                           // stages ladder 1
        auto f = index.find(kk);
        if (f != index.end()) child = f->second;
      }
      next.push_back(child);
    }
    pop.swap(next);
  }
  if (best < 0) return -1;
  if (best_out) *best_out = space[best];
  if (log) log->best_measured = best_t;
  return 0;
}

}  // namespace mbci
