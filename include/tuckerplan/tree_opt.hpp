// tuckerplan (B200 engine) : minimum-cost tree search — drop-in for reference tree_opt.hpp:120-150.
// (The exhaustive enumerator / counter of the reference, :152-279, is its test oracle and is not part of this path.)
#pragma once

#include "tree_cost.hpp"

namespace tuckerplan {

struct OptimalTreeResult {
  TtmTree tree;
  u64 total_macs = 0;
  std::size_t dp_states = 0;
};

inline OptimalTreeResult optimal_tree(const ProblemSpec& s) {
  if (s.K.size() != s.L.size()) fail(Errc::bad_dims, "spec needs matching non-empty L and K");
  OptimalTreeResult r;
  u64 states = 0;
  r.tree = detail::tree_from_abi(s.n_modes(), [&](int cap, int* k, int* m, int* p, int* n) {
    return tp_optimal_tree(s.n_modes(), s.L.data(), s.K.data(), cap, k, m, p, n, &r.total_macs, &states);
  });
  r.dp_states = static_cast<std::size_t>(states);
  return r;
}

inline u64 optimal_cost_reuse_greedy(const ProblemSpec& s) {
  if (s.K.size() != s.L.size()) fail(Errc::bad_dims, "spec needs matching non-empty L and K");
  u64 cost = 0;
  detail::check(tp_reuse_greedy_cost(s.n_modes(), s.L.data(), s.K.data(), &cost));
  return cost;
}

}  // namespace tuckerplan
