// TEST INFRASTRUCTURE — not part of the product.
//
// C entry points around the reference's own Eigen-free headers, compiled from where they lie under
// /root/reference/proj/include (nothing is copied) by oracle/Makefile into oracle/_ref/libref_shim.so.
// bench.py's `--impl reference` arm and the tests load it with ctypes so that the reference arm takes its inputs
// and selections from the reference's code only, without mapping the product library:
//   ref_random_tensor      — random_tensor(dims, seed)                       dense_tensor.hpp:43-49
//   ref_gaussians          — mt19937_64(seed) through ONE normal_distribution  hooi.hpp:111-116 (the stream only;
//                            hooi.hpp itself needs Eigen and cannot be compiled here)
//   ref_optimal_tree       — optimal_tree(spec)                              tree_opt.hpp:126-138
//   ref_tree_cost          — tree_cost / node_cardinalities                  tree_cost.hpp:25-63
//   ref_optimal_static_grid, ref_static_volume                               grid_volume.hpp:32-110
#include <cstddef>
#include <cstdint>
#include <random>
#include <vector>

#include "tuckerplan/dense_tensor.hpp"
#include "tuckerplan/grid.hpp"
#include "tuckerplan/grid_volume.hpp"
#include "tuckerplan/tree_cost.hpp"
#include "tuckerplan/tree_opt.hpp"

namespace tp = tuckerplan;
using tp::u64;

namespace {

tp::ProblemSpec spec_of(int n, const u64* L, const u64* K) {
  return tp::ProblemSpec{std::vector<u64>(L, L + n), std::vector<u64>(K, K + n)};
}

tp::TtmTree tree_of(int n_modes, int n_nodes, const int* kind, const int* mode, const int* parent) {
  tp::TtmTree t;
  t.n_modes = n_modes;
  t.nodes.resize(static_cast<std::size_t>(n_nodes));
  for (int i = 0; i < n_nodes; ++i) {
    t.nodes[i].kind = static_cast<tp::NodeKind>(kind[i]);
    t.nodes[i].mode = mode[i];
    t.nodes[i].parent = parent[i];
    if (parent[i] >= 0) t.nodes[parent[i]].children.push_back(i);
  }
  return t;
}

template <class Body>
int guarded(Body&& body) {
  try {
    body();
    return 0;
  } catch (const tp::Error& e) {
    return static_cast<int>(e.code()) + 1;
  } catch (...) {
    return 1000;
  }
}

}  // namespace

extern "C" {

int ref_random_tensor(int n_modes, const std::size_t* dims, u64 seed, double* out) {
  return guarded([&] {
    // the reference returns the tensor by value; same generator, same order, written where the caller wants it
    const tp::DenseTensor t = tp::random_tensor(std::vector<std::size_t>(dims, dims + n_modes), seed);
    for (std::size_t i = 0; i < t.data.size(); ++i) out[i] = t.data[i];
  });
}

int ref_gaussians(u64 seed, std::size_t count, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> normal(0.0, 1.0);
  for (std::size_t i = 0; i < count; ++i) out[i] = normal(rng);
  return 0;
}

int ref_optimal_tree(int n_modes, const u64* L, const u64* K, int cap, int* kind, int* mode, int* parent,
                     int* n_nodes, u64* total_macs) {
  return guarded([&] {
    const tp::OptimalTreeResult r = tp::optimal_tree(spec_of(n_modes, L, K));
    const int n = static_cast<int>(r.tree.nodes.size());
    if (n > cap) throw tp::Error(tp::Errc::bad_argument, "capacity");
    for (int i = 0; i < n; ++i) {
      kind[i] = static_cast<int>(r.tree.nodes[i].kind);
      mode[i] = r.tree.nodes[i].mode;
      parent[i] = r.tree.nodes[i].parent;
    }
    *n_nodes = n;
    if (total_macs) *total_macs = r.total_macs;
  });
}

int ref_tree_cost(int n_modes, const u64* L, const u64* K, int n_nodes, const int* kind, const int* mode,
                  const int* parent, u64* total_macs, u64* card_in, u64* card_out, int* depth) {
  return guarded([&] {
    const tp::ProblemSpec s = spec_of(n_modes, L, K);
    const tp::TtmTree t = tree_of(n_modes, n_nodes, kind, mode, parent);
    tp::validate_tree(t, s);
    const tp::CostReport c = tp::tree_cost(t, s);
    const tp::NodeCards cards = tp::node_cardinalities(t, s);
    if (total_macs) *total_macs = c.total_macs;
    if (depth) *depth = c.depth;
    for (int i = 0; i < n_nodes; ++i) {
      if (card_in) card_in[i] = cards.in[i];
      if (card_out) card_out[i] = cards.out[i];
    }
  });
}

int ref_optimal_static_grid(int n_modes, const u64* L, const u64* K, int n_nodes, const int* kind, const int* mode,
                            const int* parent, u64 procs, u64* q_out, u64* total) {
  return guarded([&] {
    const tp::ProblemSpec s = spec_of(n_modes, L, K);
    const tp::StaticGridResult r = tp::optimal_static_grid(tree_of(n_modes, n_nodes, kind, mode, parent), s, procs);
    for (int m = 0; m < n_modes; ++m) q_out[m] = r.grid.q[m];
    if (total) *total = r.report.total;
  });
}

int ref_static_volume(int n_modes, const u64* L, const u64* K, int n_nodes, const int* kind, const int* mode,
                      const int* parent, const u64* q, u64 procs, u64* total) {
  return guarded([&] {
    const tp::ProblemSpec s = spec_of(n_modes, L, K);
    tp::Grid g;
    g.q.assign(q, q + n_modes);
    *total = tp::static_volume(tree_of(n_modes, n_nodes, kind, mode, parent), s, g, procs).total;
  });
}

}  // extern "C"
