// tuckerplan (B200 engine) : communication volume under one grid — drop-in for reference grid_volume.hpp:20-110.
#pragma once

#include <vector>

#include "grid.hpp"
#include "tree_cost.hpp"

namespace tuckerplan {

struct NodeVolume {
  int node = -1;
  u64 ttm = 0;
  u64 regrid = 0;
};

struct VolumeReport {
  u64 total = 0;
  std::vector<NodeVolume> per_node;  // internal nodes in id order
};

namespace detail {
inline VolumeReport volume_report(const TtmTree& t, u64 total, const std::vector<u64>& per_node) {
  VolumeReport r;
  r.total = total;
  for (std::size_t id = 0; id < t.nodes.size(); ++id)
    if (t.is_internal(static_cast<int>(id))) r.per_node.push_back(NodeVolume{static_cast<int>(id), per_node[id], 0});
  return r;
}
}  // namespace detail

inline VolumeReport static_volume(const TtmTree& t, const ProblemSpec& s, const Grid& g, u64 procs) {
  validate_grid(g, s, procs);
  if (t.n_modes != s.n_modes()) fail(Errc::shape_mismatch, "tree and spec mode counts differ");
  const detail::FlatTree f = detail::flatten(t);
  std::vector<u64> per(f.size());
  u64 total = 0;
  detail::check(tp_static_volume(s.n_modes(), s.L.data(), s.K.data(), f.size(), f.kind.data(), f.mode.data(),
                                 f.parent.data(), g.q.data(), procs, &total, per.data()));
  return detail::volume_report(t, total, per);
}

struct StaticGridResult {
  Grid grid;
  VolumeReport report;
};

inline StaticGridResult optimal_static_grid(const TtmTree& t, const ProblemSpec& s, u64 procs, int threads = 1) {
  if (t.n_modes != s.n_modes()) fail(Errc::shape_mismatch, "tree and spec mode counts differ");
  const detail::FlatTree f = detail::flatten(t);
  std::vector<u64> per(f.size());
  StaticGridResult r;
  r.grid.q.resize(s.n_modes());
  u64 total = 0;
  detail::check(tp_optimal_static_grid(s.n_modes(), s.L.data(), s.K.data(), f.size(), f.kind.data(), f.mode.data(),
                                       f.parent.data(), procs, threads, r.grid.q.data(), &total, per.data()));
  r.report = detail::volume_report(t, total, per);
  return r;
}

}  // namespace tuckerplan
