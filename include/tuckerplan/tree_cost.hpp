// tuckerplan (B200 engine) : tree cost model — drop-in for reference tree_cost.hpp:20-86.
#pragma once

#include <vector>

#include "ttm_tree.hpp"

namespace tuckerplan {

struct NodeCards {
  std::vector<u64> in;
  std::vector<u64> out;
};

struct CostReport {
  u64 total_macs = 0;
  std::vector<u64> per_node_macs;
  int n_internal = 0;
  int depth = 0;
};

namespace detail {
inline CostReport cost_and_cards(const TtmTree& t, const ProblemSpec& s, NodeCards* cards) {
  if (t.n_modes != s.n_modes()) fail(Errc::shape_mismatch, "tree and spec mode counts differ");
  const FlatTree f = flatten(t);
  CostReport r;
  r.per_node_macs.resize(f.size());
  NodeCards c;
  c.in.resize(f.size());
  c.out.resize(f.size());
  check(tp_tree_cost(s.n_modes(), s.L.data(), s.K.data(), f.size(), f.kind.data(), f.mode.data(), f.parent.data(),
                     &r.total_macs, r.per_node_macs.data(), c.in.data(), c.out.data(), &r.n_internal, &r.depth));
  if (cards) *cards = std::move(c);
  return r;
}
}  // namespace detail

inline NodeCards node_cardinalities(const TtmTree& t, const ProblemSpec& s) {
  NodeCards c;
  detail::cost_and_cards(t, s, &c);
  return c;
}
inline CostReport tree_cost(const TtmTree& t, const ProblemSpec& s) { return detail::cost_and_cards(t, s, nullptr); }
inline u64 tree_cost_total(const TtmTree& t, const ProblemSpec& s) { return tree_cost(t, s).total_macs; }

}  // namespace tuckerplan
