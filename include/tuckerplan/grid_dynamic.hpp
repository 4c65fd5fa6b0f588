// tuckerplan (B200 engine) : per-node grid assignment — drop-in for reference grid_dynamic.hpp:32-167
// (scheme_volume, optimal_dynamic_scheme; the exhaustive brute_force_dynamic test oracle is not provided).
#pragma once

#include <map>
#include <string>
#include <vector>

#include "grid.hpp"
#include "grid_volume.hpp"
#include "tree_cost.hpp"
#include "ttm_tree.hpp"

namespace tuckerplan {

struct DynamicGridScheme {
  Grid root;
  std::map<int, Grid> node_grids;  // one entry per internal node
};

namespace detail {
// node-id-major n_nodes x n_modes table the C ABI takes; throws missing_assignment like the reference does
inline std::vector<u64> scheme_table(const TtmTree& t, int n_modes, const DynamicGridScheme& scheme) {
  std::vector<u64> flat(t.nodes.size() * static_cast<std::size_t>(n_modes), 0);
  for (std::size_t id = 0; id < t.nodes.size(); ++id) {
    if (!t.is_internal(static_cast<int>(id))) continue;
    const auto it = scheme.node_grids.find(static_cast<int>(id));
    if (it == scheme.node_grids.end()) fail(Errc::missing_assignment, "no grid for internal node " + std::to_string(id));
    if (static_cast<int>(it->second.q.size()) != n_modes) fail(Errc::invalid_grid, "grid length differs from mode count");
    for (int m = 0; m < n_modes; ++m) flat[id * n_modes + m] = it->second.q[m];
  }
  return flat;
}

inline VolumeReport scheme_report(const TtmTree& t, u64 total, const std::vector<u64>& ttm, const std::vector<u64>& regrid) {
  VolumeReport r;
  r.total = total;
  for (std::size_t id = 0; id < t.nodes.size(); ++id)
    if (t.is_internal(static_cast<int>(id)))
      r.per_node.push_back(NodeVolume{static_cast<int>(id), ttm[id], regrid[id]});
  return r;
}
}  // namespace detail

inline VolumeReport scheme_volume(const TtmTree& t, const ProblemSpec& s, const DynamicGridScheme& scheme, u64 procs) {
  validate_grid(scheme.root, s, procs);
  if (t.n_modes != s.n_modes()) fail(Errc::shape_mismatch, "tree and spec mode counts differ");
  const detail::FlatTree f = detail::flatten(t);
  const std::vector<u64> table = detail::scheme_table(t, s.n_modes(), scheme);
  std::vector<u64> ttm(f.size()), regrid(f.size());
  u64 total = 0;
  detail::check(tp_scheme_volume(s.n_modes(), s.L.data(), s.K.data(), f.size(), f.kind.data(), f.mode.data(),
                                 f.parent.data(), scheme.root.q.data(), table.data(), procs, &total, ttm.data(),
                                 regrid.data()));
  return detail::scheme_report(t, total, ttm, regrid);
}

struct DynamicOptions {
  bool legacy_regrid_target = false;  // pick the regrid grid by the children's volume alone
};

struct DynamicSchemeResult {
  DynamicGridScheme scheme;
  VolumeReport report;
};

inline DynamicSchemeResult optimal_dynamic_scheme(const TtmTree& t, const ProblemSpec& s, u64 procs,
                                                  DynamicOptions opts = {}) {
  if (t.n_modes != s.n_modes()) fail(Errc::shape_mismatch, "tree and spec mode counts differ");
  const detail::FlatTree f = detail::flatten(t);
  const int n = s.n_modes();
  std::vector<u64> root(n), table(static_cast<std::size_t>(f.size()) * n), ttm(f.size()), regrid(f.size());
  u64 total = 0;
  detail::check(tp_optimal_dynamic_scheme(n, s.L.data(), s.K.data(), f.size(), f.kind.data(), f.mode.data(),
                                          f.parent.data(), procs, opts.legacy_regrid_target ? 1 : 0, root.data(),
                                          table.data(), &total, ttm.data(), regrid.data()));
  DynamicSchemeResult r;
  r.scheme.root.q = root;
  for (std::size_t id = 0; id < t.nodes.size(); ++id)
    if (t.is_internal(static_cast<int>(id)))
      r.scheme.node_grids[static_cast<int>(id)].q.assign(table.begin() + id * n, table.begin() + (id + 1) * n);
  r.report = detail::scheme_report(t, total, ttm, regrid);
  return r;
}

}  // namespace tuckerplan
