// Compile-time pin of the API surface this repo provides under the reference's header names: every supported
// entry point is named with the reference's signature (Matrix standing in for Eigen::MatrixXd).  What is NOT here is
// not provided: bench.hpp's corpus statistics (BenchParams, generate_benchmark, run_comparison, percentile,
// reference_datasets, spec_id) and the CLI's `bench` subcommand, the tree enumerator / counter of
// tree_opt.hpp:152-279, brute_force_dynamic -- planner-side test oracles and statistics off the HOOI hot path
// (DESIGN.md §7).  Compiling this file is the test; it is never linked against a GPU.
#include <cstddef>
#include <string>
#include <vector>

#include "tuckerplan/tuckerplan.hpp"

#if __has_include("tuckerplan/bench.hpp")
#error "bench.hpp appeared: move its entry points into the pinned surface below"
#endif

namespace tp = tuckerplan;
using tp::u64;

template <class F>
constexpr bool pinned(F) {
  return true;
}

// core model
static_assert(pinned<void (*)(const tp::ProblemSpec&)>(&tp::validate_spec));
static_assert(pinned<u64 (*)(const tp::ProblemSpec&)>(&tp::input_cardinality));
static_assert(pinned<u64 (*)(const tp::ProblemSpec&)>(&tp::core_cardinality));
// trees
static_assert(pinned<void (*)(const tp::TtmTree&, const tp::ProblemSpec&)>(&tp::validate_tree));
static_assert(pinned<bool (*)(const tp::TtmTree&)>(&tp::is_canonical));
static_assert(pinned<tp::TtmTree (*)(const tp::TtmTree&)>(&tp::canonicalize));
static_assert(pinned<int (*)(const tp::TtmTree&)>(&tp::tree_depth));
static_assert(pinned<tp::NodeCards (*)(const tp::TtmTree&, const tp::ProblemSpec&)>(&tp::node_cardinalities));
static_assert(pinned<tp::CostReport (*)(const tp::TtmTree&, const tp::ProblemSpec&)>(&tp::tree_cost));
static_assert(pinned<tp::OptimalTreeResult (*)(const tp::ProblemSpec&)>(&tp::optimal_tree));
static_assert(pinned<u64 (*)(const tp::ProblemSpec&)>(&tp::optimal_cost_reuse_greedy));
static_assert(pinned<tp::TtmTree (*)(const tp::ProblemSpec&, tp::ChainOrder)>(&tp::chain_tree));
static_assert(pinned<tp::TtmTree (*)(const tp::ProblemSpec&)>(&tp::balanced_tree));
static_assert(pinned<tp::TtmTree (*)(const tp::ProblemSpec&, tp::TreeStrategy)>(&tp::build_tree));
static_assert(pinned<const char* (*)(tp::TreeStrategy)>(&tp::strategy_name));
// grids
static_assert(pinned<void (*)(const tp::Grid&, const tp::ProblemSpec&, u64)>(&tp::validate_grid));
static_assert(pinned<u64 (*)(u64, int)>(&tp::grid_count));
static_assert(pinned<std::vector<tp::Grid> (*)(u64, const tp::ProblemSpec&)>(&tp::enumerate_grids));
static_assert(pinned<std::vector<u64> (*)(u64, u64)>(&tp::block_bounds));
static_assert(pinned<u64 (*)(u64, u64, u64)>(&tp::block_of));
static_assert(pinned<tp::VolumeReport (*)(const tp::TtmTree&, const tp::ProblemSpec&, const tp::Grid&, u64)>(&tp::static_volume));
static_assert(pinned<tp::VolumeReport (*)(const tp::TtmTree&, const tp::ProblemSpec&, const tp::DynamicGridScheme&, u64)>(
    &tp::scheme_volume));
static_assert(pinned<tp::DynamicGridScheme (*)(const tp::TtmTree&, const tp::Grid&)>(&tp::uniform_scheme));
static_assert(pinned<tp::SimLedger (*)(const tp::TtmTree&, const tp::ProblemSpec&, const tp::DynamicGridScheme&, u64, bool)>(
    &tp::simulate_distribution));
// dense data and the engine
static_assert(pinned<tp::DenseTensor (*)(std::vector<std::size_t>)>(&tp::zeros));
static_assert(pinned<tp::DenseTensor (*)(std::vector<std::size_t>, std::uint64_t)>(&tp::random_tensor));
static_assert(pinned<double (*)(const tp::DenseTensor&)>(&tp::frobenius_norm));
// formats
static_assert(pinned<tp::json (*)(const tp::ProblemSpec&)>(&tp::spec_to_json));
static_assert(pinned<tp::ProblemSpec (*)(const tp::json&)>(&tp::spec_from_json));
static_assert(pinned<tp::json (*)(const tp::TtmTree&)>(&tp::tree_to_json));
static_assert(pinned<tp::TtmTree (*)(const tp::json&)>(&tp::tree_from_json));
static_assert(pinned<tp::json (*)(const tp::Grid&)>(&tp::grid_to_json));
static_assert(pinned<tp::Grid (*)(const tp::json&)>(&tp::grid_from_json));
static_assert(pinned<tp::json (*)(const tp::DynamicGridScheme&)>(&tp::scheme_to_json));
static_assert(pinned<tp::DynamicGridScheme (*)(const tp::json&)>(&tp::scheme_from_json));
static_assert(pinned<tp::json (*)(const tp::CostReport&)>(&tp::cost_to_json));
static_assert(pinned<tp::json (*)(const tp::VolumeReport&)>(&tp::volume_to_json));
static_assert(pinned<tp::json (*)(const tp::SimLedger&)>(&tp::ledger_to_json));
static_assert(pinned<void (*)(const std::string&, const tp::DenseTensor&)>(&tp::write_tensor));
static_assert(pinned<tp::DenseTensor (*)(const std::string&)>(&tp::read_tensor));

// templates and defaulted arguments: named in (uninstantiated-at-run-time) code so that they must at least resolve
[[maybe_unused]] static void engine_surface(const tp::DenseTensor& t, const tp::ProblemSpec& s, const tp::TtmTree& tree,
                                            const tp::Matrix& m, tp::Decomposition d) {
  tp::u64 macs = 0;
  tp::SweepStats stats;
  (void)tp::ttm(t, m, 0, &macs);
  (void)tp::unfold(t, 0);
  (void)tp::fold(m, t.dims, 0);
  (void)tp::leading_left_factors(m, 1);
  (void)tp::random_decomposition(t, s, 0);
  d = tp::hooi_sweep(t, s, d, tree, tp::SweepKind::jacobi, &stats);
  d = tp::hooi_sweep(t, s, d, tree, tp::SweepKind::gauss_seidel);
  (void)tp::reconstruction_error(t, d);
  (void)tp::optimal_static_grid(tree, s, 2);
  (void)tp::optimal_dynamic_scheme(tree, s, 2);
  (void)tp::sthosvd(t, s);
  tp::DeviceHooi resident(t, s, tree, tp::SweepKind::jacobi);
  tp::GridHooi grid(t, s, tree, tp::uniform_scheme(tree, tp::Grid{{1}}), {0});
  (void)tp::tol::kProjectorTol;
  (void)tp::kMaxGramRows;
}

int main() { return 0; }
