// tuckerplan (B200 engine) : chain and balanced trees — drop-in for reference tree_builders.hpp:25-91, plus the
// strategy switch of bench.hpp:115-139.
#pragma once

#include "tree_opt.hpp"

namespace tuckerplan {

enum class ChainOrder { input, by_cost, by_ratio };

inline TtmTree chain_tree(const ProblemSpec& s, ChainOrder ord = ChainOrder::input) {
  if (s.K.size() != s.L.size()) fail(Errc::bad_dims, "spec needs matching non-empty L and K");
  return detail::tree_from_abi(s.n_modes(), [&](int cap, int* k, int* m, int* p, int* n) {
    return tp_chain_tree(s.n_modes(), s.L.data(), s.K.data(), static_cast<int>(ord), cap, k, m, p, n);
  });
}

inline TtmTree balanced_tree(const ProblemSpec& s) {
  if (s.K.size() != s.L.size()) fail(Errc::bad_dims, "spec needs matching non-empty L and K");
  return detail::tree_from_abi(s.n_modes(), [&](int cap, int* k, int* m, int* p, int* n) {
    return tp_balanced_tree(s.n_modes(), s.L.data(), s.K.data(), cap, k, m, p, n);
  });
}

enum class TreeStrategy { chain_input, chain_by_cost, chain_by_ratio, balanced, optimal };

inline const char* strategy_name(TreeStrategy s) {
  static const char* const names[] = {"chain-input", "chain-k", "chain-h", "balanced", "opt"};
  return names[static_cast<int>(s)];
}

inline TtmTree build_tree(const ProblemSpec& s, TreeStrategy strategy) {
  if (s.K.size() != s.L.size()) fail(Errc::bad_dims, "spec needs matching non-empty L and K");
  return detail::tree_from_abi(s.n_modes(), [&](int cap, int* k, int* m, int* p, int* n) {
    return tp_build_tree(s.n_modes(), s.L.data(), s.K.data(), static_cast<int>(strategy), cap, k, m, p, n);
  });
}

}  // namespace tuckerplan
