// TEST INFRASTRUCTURE — not part of the product.
//
// Driver around the reference's own Eigen-free headers (compiled from where
// they lie under /root/reference/proj/include; nothing is copied).  Built by
// oracle/Makefile into oracle/_ref/ref_tools.  It exposes, as JSON on stdout
// or raw little-endian f64 files:
//   plan      — optimal_tree / chain_tree / balanced_tree / tree_cost /
//               node_cardinalities / enumerate_grids / optimal_static_grid /
//               static_volume / count_reduce_scatter   (planner goldens)
//   tensor    — random_tensor(dims, seed)                (dense_tensor.hpp:43-49)
//   gaussians — the first `count` draws of mt19937_64(seed) through ONE
//               std::normal_distribution<double> object, i.e. the stream
//               random_decomposition consumes (hooi.hpp:111-116; hooi.hpp
//               itself needs Eigen and cannot be compiled here)
//   blocks    — block_bounds / block_of                  (grid.hpp:114-125)
//   psi       — grid_count                                (grid.hpp:49-70)
//   dynamic   — optimal_dynamic_scheme (both objectives) / scheme_volume / simulate_distribution in trace mode
//               where its guards allow (grid_dynamic.hpp:141-167, simulate.hpp:123-178)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "tuckerplan/dense_tensor.hpp"
#include "tuckerplan/grid.hpp"
#include "tuckerplan/grid_volume.hpp"
#include "tuckerplan/grid_dynamic.hpp"
#include "tuckerplan/simulate.hpp"
#include "tuckerplan/tree_builders.hpp"
#include "tuckerplan/tree_cost.hpp"
#include "tuckerplan/tree_opt.hpp"

namespace tp = tuckerplan;
using tp::u64;

static std::vector<u64> parse_list(const char* s) {
  std::vector<u64> v;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ',')) v.push_back(std::strtoull(item.c_str(), nullptr, 10));
  return v;
}

template <class T>
static std::string arr(const std::vector<T>& v) {
  std::string s = "[";
  for (std::size_t i = 0; i < v.size(); ++i) {
    if (i) s += ",";
    s += std::to_string(v[i]);
  }
  return s + "]";
}

static std::string tree_json(const tp::TtmTree& t, const tp::ProblemSpec& s) {
  std::vector<int> kind, mode, parent;
  for (const auto& n : t.nodes) {
    kind.push_back(static_cast<int>(n.kind));
    mode.push_back(n.mode);
    parent.push_back(n.parent);
  }
  const tp::CostReport c = tp::tree_cost(t, s);
  const tp::NodeCards cards = tp::node_cardinalities(t, s);
  std::string out = "{\"kind\":" + arr(kind) + ",\"mode\":" + arr(mode) + ",\"parent\":" + arr(parent);
  out += ",\"total_macs\":" + std::to_string(c.total_macs) + ",\"per_node_macs\":" + arr(c.per_node_macs);
  out += ",\"n_internal\":" + std::to_string(c.n_internal) + ",\"depth\":" + std::to_string(c.depth);
  out += ",\"canonical\":" + std::string(tp::is_canonical(t) ? "true" : "false");
  out += ",\"card_in\":" + arr(cards.in) + ",\"card_out\":" + arr(cards.out) + "}";
  return out;
}

static int cmd_plan(int argc, char** argv) {
  if (argc < 4) return 2;
  tp::ProblemSpec s{parse_list(argv[2]), parse_list(argv[3])};
  std::vector<u64> procs = argc > 4 ? parse_list(argv[4]) : std::vector<u64>{};
  try {
    const tp::OptimalTreeResult opt = tp::optimal_tree(s);
    std::string out = "{\"L\":" + arr(s.L) + ",\"K\":" + arr(s.K);
    out += ",\"opt\":" + tree_json(opt.tree, s) + ",\"opt_total_macs\":" + std::to_string(opt.total_macs);
    out += ",\"dp_states\":" + std::to_string(opt.dp_states);
    out += ",\"reuse_greedy_macs\":" + std::to_string(tp::optimal_cost_reuse_greedy(s));
    out += ",\"chain_input\":" + tree_json(tp::chain_tree(s, tp::ChainOrder::input), s);
    out += ",\"chain_by_cost\":" + tree_json(tp::chain_tree(s, tp::ChainOrder::by_cost), s);
    out += ",\"chain_by_ratio\":" + tree_json(tp::chain_tree(s, tp::ChainOrder::by_ratio), s);
    out += ",\"balanced\":" + tree_json(tp::balanced_tree(s), s);
    out += ",\"canonical_chain\":" + tree_json(tp::canonicalize(tp::chain_tree(s)), s);
    out += ",\"grids\":{";
    bool first = true;
    for (u64 p : procs) {
      if (!first) out += ",";
      first = false;
      out += "\"" + std::to_string(p) + "\":{";
      const std::vector<tp::Grid> grids = tp::enumerate_grids(p, s);
      out += "\"enumerated\":[";
      for (std::size_t i = 0; i < grids.size(); ++i) out += (i ? "," : "") + arr(grids[i].q);
      out += "]";
      if (!grids.empty()) {
        const tp::StaticGridResult r = tp::optimal_static_grid(opt.tree, s, p);
        std::vector<u64> per;
        std::vector<int> ids;
        std::vector<u64> traced;
        for (const auto& nv : r.report.per_node) {
          per.push_back(nv.ttm);
          ids.push_back(nv.node);
          traced.push_back(tp::detail::count_reduce_scatter(
              tp::detail::node_extents(opt.tree, s, nv.node), r.grid, opt.tree.nodes[nv.node].mode));
        }
        out += ",\"best\":" + arr(r.grid.q) + ",\"best_volume\":" + std::to_string(r.report.total);
        out += ",\"per_node_ids\":" + arr(ids) + ",\"per_node_ttm\":" + arr(per) + ",\"traced_ttm\":" + arr(traced);
        std::vector<u64> vols;
        for (const auto& g : grids) vols.push_back(tp::static_volume(opt.tree, s, g, p).total);
        out += ",\"volumes\":" + arr(vols);
      }
      out += "}";
    }
    out += "}}";
    std::puts(out.c_str());
  } catch (const tp::Error& e) {
    std::printf("{\"L\":%s,\"K\":%s,\"error\":%d,\"error_mode\":%d}\n", arr(s.L).c_str(), arr(s.K).c_str(),
                static_cast<int>(e.code()), e.mode());
  }
  return 0;
}

static tp::TtmTree tree_by_name(const std::string& name, const tp::ProblemSpec& s) {
  if (name == "opt") return tp::optimal_tree(s).tree;
  if (name == "chain") return tp::chain_tree(s, tp::ChainOrder::input);
  if (name == "chain_by_cost") return tp::chain_tree(s, tp::ChainOrder::by_cost);
  if (name == "balanced") return tp::balanced_tree(s);
  throw tp::Error(tp::Errc::bad_argument, "unknown tree name");
}

static std::string scheme_json(const tp::TtmTree& t, const tp::ProblemSpec& s, const tp::DynamicSchemeResult& r,
                               u64 procs) {
  std::string out = "{\"root\":" + arr(r.scheme.root.q) + ",\"total\":" + std::to_string(r.report.total);
  std::vector<int> ids;
  std::vector<u64> ttm, regrid;
  std::string grids = "[";
  for (const auto& nv : r.report.per_node) {
    if (!ids.empty()) grids += ",";
    ids.push_back(nv.node);
    ttm.push_back(nv.ttm);
    regrid.push_back(nv.regrid);
    grids += arr(r.scheme.node_grids.at(nv.node).q);
  }
  out += ",\"nodes\":" + arr(ids) + ",\"node_grids\":" + grids + "]";
  out += ",\"ttm\":" + arr(ttm) + ",\"regrid\":" + arr(regrid);
  if (tp::input_cardinality(s) <= tp::kTraceMaxElements && procs <= tp::kTraceMaxProcs) {
    const tp::SimLedger led = tp::simulate_distribution(t, s, r.scheme, procs, true);
    std::vector<u64> mt, mr;
    for (const auto& nt : led.nodes) {
      mt.push_back(nt.measured_ttm);
      mr.push_back(nt.measured_regrid);
    }
    out += ",\"traced_ttm\":" + arr(mt) + ",\"traced_regrid\":" + arr(mr);
  }
  return out + "}";
}

static int cmd_dynamic(int argc, char** argv) {
  if (argc < 6) return 2;
  tp::ProblemSpec s{parse_list(argv[2]), parse_list(argv[3])};
  const u64 procs = std::strtoull(argv[4], nullptr, 10);
  const std::string name = argv[5];
  try {
    const tp::TtmTree t = tree_by_name(name, s);
    std::string out = "{\"L\":" + arr(s.L) + ",\"K\":" + arr(s.K) + ",\"procs\":" + std::to_string(procs);
    out += ",\"tree_name\":\"" + name + "\",\"tree\":" + tree_json(t, s);
    tp::DynamicOptions legacy;
    legacy.legacy_regrid_target = true;
    out += ",\"scheme\":" + scheme_json(t, s, tp::optimal_dynamic_scheme(t, s, procs), procs);
    out += ",\"legacy\":" + scheme_json(t, s, tp::optimal_dynamic_scheme(t, s, procs, legacy), procs);
    out += ",\"static_total\":" + std::to_string(tp::optimal_static_grid(t, s, procs).report.total);
    std::puts((out + "}").c_str());
  } catch (const tp::Error& e) {
    std::printf("{\"L\":%s,\"K\":%s,\"procs\":%llu,\"tree_name\":\"%s\",\"error\":%d}\n", arr(s.L).c_str(),
                arr(s.K).c_str(), (unsigned long long)procs, name.c_str(), static_cast<int>(e.code()));
  }
  return 0;
}

static int write_raw(const char* path, const std::vector<double>& v) {
  FILE* f = std::fopen(path, "wb");
  if (!f) return 1;
  std::fwrite(v.data(), sizeof(double), v.size(), f);
  std::fclose(f);
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string cmd = argv[1];
  if (cmd == "plan") return cmd_plan(argc, argv);
  if (cmd == "dynamic") return cmd_dynamic(argc, argv);
  if (cmd == "tensor" && argc == 5) {
    const std::vector<u64> d = parse_list(argv[2]);
    const tp::DenseTensor t =
        tp::random_tensor(std::vector<std::size_t>(d.begin(), d.end()), std::strtoull(argv[3], nullptr, 10));
    return write_raw(argv[4], t.data);
  }
  if (cmd == "gaussians" && argc == 5) {
    const u64 count = std::strtoull(argv[2], nullptr, 10);
    std::mt19937_64 rng(std::strtoull(argv[3], nullptr, 10));
    std::normal_distribution<double> normal(0.0, 1.0);
    std::vector<double> v(count);
    for (double& x : v) x = normal(rng);
    return write_raw(argv[4], v);
  }
  if (cmd == "blocks" && argc == 4) {
    const u64 len = std::strtoull(argv[2], nullptr, 10), parts = std::strtoull(argv[3], nullptr, 10);
    std::vector<u64> owner;
    for (u64 c = 0; c < len; ++c) owner.push_back(tp::block_of(c, len, parts));
    std::printf("{\"len\":%llu,\"parts\":%llu,\"cuts\":%s,\"block_of\":%s}\n", (unsigned long long)len,
                (unsigned long long)parts, arr(tp::block_bounds(len, parts)).c_str(), arr(owner).c_str());
    return 0;
  }
  if (cmd == "psi" && argc == 4) {
    std::printf("%llu\n", (unsigned long long)tp::grid_count(std::strtoull(argv[2], nullptr, 10), std::atoi(argv[3])));
    return 0;
  }
  return 2;
}
