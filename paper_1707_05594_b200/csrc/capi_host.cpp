// extern "C" surface for the host-only part of the library: planner and
// seeded input generation.  See include/tuckerplan_b200.h for the contract.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"
#include "hostgen.hpp"
#include "planner.hpp"

namespace tpb {
namespace {
thread_local std::string g_error_text;
thread_local int g_error_mode = -1;
}  // namespace

void set_last_error(int /*status*/, const std::string& what, int mode) {
  g_error_text = what;
  g_error_mode = mode;
}

namespace {
void export_tree(const Tree& t, int cap, int* kind, int* mode, int* parent, int* n_nodes) {
  if (n_nodes) *n_nodes = t.size();
  if (t.size() > cap) raise(TP_ERR_CAPACITY, "tree has " + std::to_string(t.size()) + " nodes, capacity too small");
  for (int i = 0; i < t.size(); ++i) {
    if (kind) kind[i] = t.kind[i];
    if (mode) mode[i] = t.mode[i];
    if (parent) parent[i] = t.parent[i];
  }
}
}  // namespace
}  // namespace tpb

using namespace tpb;

extern "C" {

const char* tp_last_error(void) { return g_error_text.c_str(); }
int tp_last_error_mode(void) { return g_error_mode; }
const char* tp_version(void) { return "tuckerplan_b200 0.1 (sm_100a)"; }

int tp_validate_spec(int n, const tp_u64* L, const tp_u64* K) {
  return guarded([&] { validate_spec(make_spec(n, L, K)); });
}

int tp_partial_cardinality(int n, const tp_u64* L, const tp_u64* K, uint32_t done, tp_u64* out) {
  return guarded([&] { *out = partial_cardinality(make_spec(n, L, K), done); });
}

int tp_optimal_tree(int n, const tp_u64* L, const tp_u64* K, int cap, int* kind, int* mode, int* parent,
                    int* n_nodes, tp_u64* total_macs, tp_u64* dp_states) {
  return guarded([&] {
    const OptimalTree r = optimal_tree(make_spec(n, L, K));
    if (total_macs) *total_macs = r.total_macs;
    if (dp_states) *dp_states = r.dp_states;
    export_tree(r.tree, cap, kind, mode, parent, n_nodes);
  });
}

int tp_reuse_greedy_cost(int n, const tp_u64* L, const tp_u64* K, tp_u64* cost) {
  return guarded([&] { *cost = reuse_greedy_cost(make_spec(n, L, K)); });
}

int tp_chain_tree(int n, const tp_u64* L, const tp_u64* K, int order, int cap, int* kind, int* mode, int* parent,
                  int* n_nodes) {
  return guarded([&] { export_tree(chain_tree(make_spec(n, L, K), order), cap, kind, mode, parent, n_nodes); });
}

int tp_balanced_tree(int n, const tp_u64* L, const tp_u64* K, int cap, int* kind, int* mode, int* parent,
                     int* n_nodes) {
  return guarded([&] { export_tree(balanced_tree(make_spec(n, L, K)), cap, kind, mode, parent, n_nodes); });
}

int tp_build_tree(int n, const tp_u64* L, const tp_u64* K, int strategy, int cap, int* kind, int* mode, int* parent,
                  int* n_nodes) {
  return guarded([&] { export_tree(build_tree(make_spec(n, L, K), strategy), cap, kind, mode, parent, n_nodes); });
}

int tp_validate_tree(int n, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind, const int* mode,
                     const int* parent) {
  return guarded([&] {
    const Spec s = make_spec(n, L, K);
    if (n_nodes <= 0 || kind[0] != TP_NODE_ROOT || parent[0] != -1) {
      if (n != s.n()) raise(TP_ERR_SHAPE_MISMATCH, "tree and spec mode counts differ");
      raise(TP_ERR_BAD_TREE, "node 0 must be the root");
    }
    validate_tree(tree_from_arrays(n, n_nodes, kind, mode, parent), s);
  });
}

int tp_tree_is_canonical(int n_nodes, const int* kind, const int* mode, const int* parent, int* out) {
  return guarded([&] { *out = is_canonical(tree_from_arrays(0, n_nodes, kind, mode, parent)) ? 1 : 0; });
}

int tp_canonicalize(int n_modes, int n_nodes, const int* kind, const int* mode, const int* parent, int cap,
                    int* out_kind, int* out_mode, int* out_parent, int* out_n_nodes) {
  return guarded([&] {
    export_tree(canonicalize(tree_from_arrays(n_modes, n_nodes, kind, mode, parent)), cap, out_kind, out_mode,
                out_parent, out_n_nodes);
  });
}

int tp_tree_depth(int n_nodes, const int* kind, const int* mode, const int* parent, int* depth) {
  return guarded([&] { *depth = tree_depth(tree_from_arrays(0, n_nodes, kind, mode, parent)); });
}

int tp_tree_cost(int n, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind, const int* mode,
                 const int* parent, tp_u64* total_macs, tp_u64* per_node_macs, tp_u64* card_in, tp_u64* card_out,
                 int* n_internal, int* depth) {
  return guarded([&] {
    const Spec s = make_spec(n, L, K);
    const Tree t = tree_from_arrays(n, n_nodes, kind, mode, parent);
    Cards cards;
    const Cost c = tree_cost(t, s, &cards);
    if (total_macs) *total_macs = c.total_macs;
    if (n_internal) *n_internal = c.n_internal;
    if (depth) *depth = c.depth;
    for (int i = 0; i < t.size(); ++i) {
      if (per_node_macs) per_node_macs[i] = c.per_node[i];
      if (card_in) card_in[i] = cards.in[i];
      if (card_out) card_out[i] = cards.out[i];
    }
  });
}

int tp_grid_count(tp_u64 procs, int n_modes, tp_u64* out) {
  return guarded([&] { *out = grid_count(procs, n_modes); });
}

int tp_validate_grid(int n, const tp_u64* L, const tp_u64* K, const tp_u64* q, tp_u64 procs) {
  return guarded([&] { validate_grid(Grid(q, q + n), make_spec(n, L, K), procs); });
}

int tp_enumerate_grids(int n, const tp_u64* L, const tp_u64* K, tp_u64 procs, size_t cap_grids, tp_u64* grids_out,
                       size_t* n_grids) {
  return guarded([&] {
    const std::vector<Grid> grids = enumerate_grids(procs, make_spec(n, L, K));
    if (n_grids) *n_grids = grids.size();
    if (grids.size() > cap_grids) raise(TP_ERR_CAPACITY, "more grids than capacity");
    for (std::size_t i = 0; i < grids.size(); ++i)
      for (int m = 0; m < n; ++m) grids_out[i * n + m] = grids[i][m];
  });
}

int tp_block_bounds(tp_u64 len, tp_u64 parts, tp_u64* cuts) {
  return guarded([&] {
    const std::vector<u64> c = block_bounds(len, parts);
    std::memcpy(cuts, c.data(), c.size() * sizeof(u64));
  });
}

int tp_block_of(tp_u64 c, tp_u64 len, tp_u64 parts, tp_u64* out) {
  return guarded([&] { *out = block_of(c, len, parts); });
}

int tp_static_volume(int n, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind, const int* mode,
                     const int* parent, const tp_u64* q, tp_u64 procs, tp_u64* total, tp_u64* per_node_ttm) {
  return guarded([&] {
    const Tree t = tree_from_arrays(n, n_nodes, kind, mode, parent);
    const Volume v = static_volume(t, make_spec(n, L, K), Grid(q, q + n), procs);
    if (total) *total = v.total;
    if (per_node_ttm) std::memcpy(per_node_ttm, v.per_node.data(), v.per_node.size() * sizeof(u64));
  });
}

int tp_optimal_static_grid(int n, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind, const int* mode,
                           const int* parent, tp_u64 procs, int threads, tp_u64* q_out, tp_u64* total,
                           tp_u64* per_node_ttm) {
  return guarded([&] {
    const Tree t = tree_from_arrays(n, n_nodes, kind, mode, parent);
    const StaticGrid g = optimal_static_grid(t, make_spec(n, L, K), procs, threads);
    for (int m = 0; m < n; ++m) q_out[m] = g.q[m];
    if (total) *total = g.volume.total;
    if (per_node_ttm) std::memcpy(per_node_ttm, g.volume.per_node.data(), g.volume.per_node.size() * sizeof(u64));
  });
}

static Scheme scheme_from_arrays(const Tree& t, int n, const tp_u64* root_grid, const tp_u64* node_grids) {
  if (!root_grid || !node_grids) raise(TP_ERR_BAD_ARGUMENT, "null grid array");
  Scheme sc;
  sc.root.assign(root_grid, root_grid + n);
  sc.node.assign(t.size(), Grid{});
  for (int id = 0; id < t.size(); ++id)
    if (t.internal(id)) sc.node[id].assign(node_grids + static_cast<size_t>(id) * n, node_grids + static_cast<size_t>(id + 1) * n);
  return sc;
}

static void scheme_volume_out(const SchemeVolume& v, tp_u64* total, tp_u64* per_node_ttm, tp_u64* per_node_regrid) {
  if (total) *total = v.total;
  if (per_node_ttm) std::memcpy(per_node_ttm, v.ttm.data(), v.ttm.size() * sizeof(u64));
  if (per_node_regrid) std::memcpy(per_node_regrid, v.regrid.data(), v.regrid.size() * sizeof(u64));
}

int tp_scheme_volume(int n, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind, const int* mode,
                     const int* parent, const tp_u64* root_grid, const tp_u64* node_grids, tp_u64 procs,
                     tp_u64* total, tp_u64* per_node_ttm, tp_u64* per_node_regrid) {
  return guarded([&] {
    const Tree t = tree_from_arrays(n, n_nodes, kind, mode, parent);
    const Scheme sc = scheme_from_arrays(t, n, root_grid, node_grids);
    scheme_volume_out(scheme_volume(t, make_spec(n, L, K), sc, procs), total, per_node_ttm, per_node_regrid);
  });
}

int tp_optimal_dynamic_scheme(int n, const tp_u64* L, const tp_u64* K, int n_nodes, const int* kind, const int* mode,
                              const int* parent, tp_u64 procs, int legacy_target, tp_u64* root_grid_out,
                              tp_u64* node_grids_out, tp_u64* total, tp_u64* per_node_ttm, tp_u64* per_node_regrid) {
  return guarded([&] {
    if (!root_grid_out || !node_grids_out) raise(TP_ERR_BAD_ARGUMENT, "null grid array");
    const Tree t = tree_from_arrays(n, n_nodes, kind, mode, parent);
    const DynamicScheme r = optimal_dynamic_scheme(t, make_spec(n, L, K), procs, legacy_target != 0);
    for (int m = 0; m < n; ++m) root_grid_out[m] = r.scheme.root[m];
    for (int id = 0; id < t.size(); ++id)
      for (int m = 0; m < n; ++m)
        node_grids_out[static_cast<size_t>(id) * n + m] = r.scheme.node[id].empty() ? 0 : r.scheme.node[id][m];
    scheme_volume_out(r.volume, total, per_node_ttm, per_node_regrid);
  });
}

int tp_count_moved(int n, const tp_u64* ext, const tp_u64* from_grid, const tp_u64* to_grid, tp_u64* out) {
  return guarded([&] {
    if (n <= 0 || !ext || !from_grid || !to_grid || !out) raise(TP_ERR_BAD_ARGUMENT, "null argument");
    for (int m = 0; m < n; ++m)
      if (ext[m] == 0 || from_grid[m] == 0 || to_grid[m] == 0) raise(TP_ERR_INVALID_GRID, "zero extent", m);
    *out = count_moved(std::vector<u64>(ext, ext + n), Grid(from_grid, from_grid + n), Grid(to_grid, to_grid + n));
  });
}

int tp_random_tensor(int n_modes, const size_t* dims, tp_u64 seed, double* out) {
  return guarded([&] {
    if (n_modes <= 0 || !dims) raise(TP_ERR_BAD_DIMS, "tensor needs at least one mode");
    std::size_t total = 1;
    for (int m = 0; m < n_modes; ++m) {
      if (dims[m] == 0) raise(TP_ERR_BAD_DIMS, "zero extent");  // zeros(), dense_tensor.hpp:35-36
      total = static_cast<std::size_t>(mul_or_throw(total, dims[m]));
    }
    GaussianStream stream(seed);
    stream.fill(out, total);
  });
}

int tp_random_orthonormal_factors(int n, const tp_u64* L, const tp_u64* K, tp_u64 seed, double* const* factors_out) {
  return guarded([&] {
    const Spec s = make_spec(n, L, K);
    validate_spec(s);
    GaussianStream stream(seed);  // ONE stream shared by all modes, hooi.hpp:111-112
    for (int m = 0; m < n; ++m) {
      const std::size_t rows = s.L[m], cols = s.K[m];
      std::vector<double> g(rows * cols);
      stream.fill(g.data(), g.size());  // column by column == column-major storage order
      householder_thin_q(g.data(), rows, cols, factors_out[m]);
    }
  });
}

int tp_frobenius_norm_host(size_t n, const double* data, double* out) {
  return guarded([&] {
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) sum += data[i] * data[i];
    *out = std::sqrt(sum);
  });
}

}  // extern "C"
