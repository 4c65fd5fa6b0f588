// A caller written against the reference's API (names as in reference tools/tuckerplan_cli.cpp:376-445 and
// tests/test_engine.cpp), compiled against include/tuckerplan/ of THIS repo and linked to libtuckerplan_b200.so.
//   dropin planner  -> planner selections for the cube / pinned specs (no GPU needed)
//   dropin hooi     -> the README transcript: 12x10x8 seed 7, K = 4,3,2, Gauss-Seidel on the chain-input tree
//   dropin grid     -> Jacobi sweeps on P = 2 and P = 4 ranks (GridHooi; virtual ranks on device 0) against the
//                      single-device DeviceHooi on the same input: projector gaps, fit, shipped volumes vs the model
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "tuckerplan/tuckerplan.hpp"

namespace tp = tuckerplan;

static std::string label(const tp::TtmTree& t, int id = 0) {
  const tp::TreeNode& n = t.nodes[id];
  std::string s = n.kind == tp::NodeKind::root ? "T" : (n.kind == tp::NodeKind::mode ? "M" : "F");
  if (n.kind != tp::NodeKind::root) s += std::to_string(n.mode + 1);
  if (!n.children.empty()) {
    s += "(";
    for (std::size_t i = 0; i < n.children.size(); ++i) s += (i ? ", " : "") + label(t, n.children[i]);
    s += ")";
  }
  return s;
}

int main(int argc, char** argv) {
  const std::string cmd = argc > 1 ? argv[1] : "planner";
  try {
    if (cmd == "planner") {
      const tp::ProblemSpec cube{{4, 4, 4}, {2, 2, 2}};
      std::printf("chain %llu\n", (unsigned long long)tp::tree_cost(tp::chain_tree(cube), cube).total_macs);
      std::printf("opt %llu\n", (unsigned long long)tp::optimal_tree(cube).total_macs);
      const tp::StaticGridResult g = tp::optimal_static_grid(tp::chain_tree(cube), cube, 4);
      std::printf("grid %llux%llux%llu vol %llu\n", (unsigned long long)g.grid.q[0], (unsigned long long)g.grid.q[1],
                  (unsigned long long)g.grid.q[2], (unsigned long long)g.report.total);
      const tp::ProblemSpec c3{{400, 100, 100, 50}, {40, 10, 20, 5}};
      std::printf("tree %s\n", label(tp::optimal_tree(c3).tree).c_str());
      std::printf("canonical %d depth %d\n", tp::is_canonical(tp::canonicalize(tp::chain_tree(cube))) ? 1 : 0,
                  tp::tree_depth(tp::optimal_tree(c3).tree));
      try {
        tp::validate_spec(tp::ProblemSpec{{3, 3}, {1, 4}});
      } catch (const tp::Error& e) {
        std::printf("error %d mode %d\n", static_cast<int>(e.code()), e.mode());
      }
      try {
        tp::optimal_static_grid(tp::chain_tree(cube), cube, 7);
      } catch (const tp::Error& e) {
        std::printf("error %d\n", static_cast<int>(e.code()));
      }
      const tp::DenseTensor t = tp::random_tensor({3, 4, 2}, 5);
      const tp::DenseTensor back = tp::fold(tp::unfold(t, 1), t.dims, 1);
      std::printf("fold %d first %.17g\n", back.data == t.data ? 1 : 0, t.data[0]);
      // per-node grids (grid_dynamic.hpp): C4 at P = 8 is where regridding pays
      const tp::ProblemSpec c4{{48, 48, 48, 48, 48}, {8, 8, 8, 8, 8}};
      const tp::TtmTree t4 = tp::optimal_tree(c4).tree;
      const tp::DynamicSchemeResult dyn = tp::optimal_dynamic_scheme(t4, c4, 8);
      int regrids = 0;
      for (const tp::NodeVolume& nv : dyn.report.per_node) regrids += nv.regrid ? 1 : 0;
      std::printf("dynamic %llu regrids %d static %llu again %llu\n", (unsigned long long)dyn.report.total, regrids,
                  (unsigned long long)tp::optimal_static_grid(t4, c4, 8).report.total,
                  (unsigned long long)tp::scheme_volume(t4, c4, dyn.scheme, 8).total);
      tp::DynamicGridScheme holes = dyn.scheme;
      holes.node_grids.erase(holes.node_grids.begin());
      try {
        tp::scheme_volume(t4, c4, holes, 8);
      } catch (const tp::Error& e) {
        std::printf("error %d\n", static_cast<int>(e.code()));
      }
      return 0;
    }
    if (cmd == "hooi") {
      const tp::DenseTensor t = tp::random_tensor({12, 10, 8}, 7);
      tp::ProblemSpec s;
      for (std::size_t d : t.dims) s.L.push_back(d);
      s.K = {4, 3, 2};
      const tp::TtmTree tree = tp::build_tree(s, tp::TreeStrategy::chain_input);
      tp::Decomposition d = tp::random_decomposition(t, s, 0);
      std::printf("start: error %.12f\n", tp::reconstruction_error(t, d));
      for (int i = 0; i < 2; ++i) {
        tp::SweepStats stats;
        d = tp::hooi_sweep(t, s, d, tree, tp::SweepKind::gauss_seidel, &stats);
        std::printf("sweep %d: error %.12f, tree macs %llu, peak live %d\n", i + 1, tp::reconstruction_error(t, d),
                    (unsigned long long)stats.tree_macs, stats.peak_live);
      }
      // the resident form gives the same numbers
      tp::DeviceHooi resident(t, s, tp::optimal_tree(s).tree, tp::SweepKind::jacobi);
      resident.set_factors(tp::random_decomposition(t, s, 0).factors);
      const tp::SweepStats st = resident.sweep();
      std::printf("resident jacobi: error %.12f, tree macs %llu\n", resident.reconstruction_error(),
                  (unsigned long long)st.tree_macs);
      try {
        tp::hooi_sweep(t, s, d, tp::balanced_tree(s), tp::SweepKind::gauss_seidel);
      } catch (const tp::Error& e) {
        std::printf("error %d\n", static_cast<int>(e.code()));
      }
      return 0;
    }
    if (cmd == "grid") {
      const tp::DenseTensor noise = tp::random_tensor({30, 24, 20}, 11);
      tp::ProblemSpec s{{30, 24, 20}, {5, 4, 3}};
      // low-rank-plus-noise input assembled with the public API: X = G x A_0 x A_1 x A_2, T = X + 1e-2 E
      const tp::Decomposition gen = tp::random_decomposition(noise, s, 3);
      tp::DenseTensor x = tp::random_tensor({5, 4, 3}, 4);
      for (int m = 0; m < 3; ++m) x = tp::ttm(x, gen.factors[m], m);
      tp::DenseTensor t = x;
      for (std::size_t i = 0; i < t.data.size(); ++i) t.data[i] += 1e-2 * noise.data[i];
      const tp::TtmTree tree = tp::optimal_tree(s).tree;
      const std::vector<tp::Matrix> start = tp::random_decomposition(t, s, 0).factors;
      tp::DeviceHooi single(t, s, tree, tp::SweepKind::jacobi);
      single.set_factors(start);
      for (int i = 0; i < 3; ++i) single.sweep();
      const tp::Decomposition want = single.decomposition();
      const double want_fit = single.reconstruction_error();
      auto projector_gap = [](const tp::Matrix& a, const tp::Matrix& b) {  // ||A A^T - B B^T||_F
        double sum = 0.0;
        for (std::size_t i = 0; i < a.rows(); ++i)
          for (std::size_t j = 0; j < a.rows(); ++j) {
            double pa = 0.0, pb = 0.0;
            for (std::size_t c = 0; c < a.cols(); ++c) {
              pa += a(i, c) * a(j, c);
              pb += b(i, c) * b(j, c);
            }
            sum += (pa - pb) * (pa - pb);
          }
        return std::sqrt(sum);
      };
      for (const tp::u64 procs : {2, 4}) {
        const tp::StaticGridResult best = tp::optimal_static_grid(tree, s, procs);
        tp::GridHooi grid(t, s, tree, tp::uniform_scheme(tree, best.grid), std::vector<int>(procs, 0));
        grid.set_factors(start);
        tp::SweepStats st;
        for (int i = 0; i < 3; ++i) st = grid.sweep();
        const tp::Decomposition got = grid.decomposition();
        double gap = 0.0;
        for (int m = 0; m < 3; ++m) gap = std::max(gap, projector_gap(got.factors[m], want.factors[m]));
        const tp::GridHooi::Volumes vol = grid.last_volumes();
        tp::u64 shipped = 0;
        for (tp::u64 v : vol.ttm) shipped += v;
        std::printf("procs %llu grid %llux%llux%llu gap_ok %d fit_ok %d macs_ok %d shipped %llu model %llu\n",
                    (unsigned long long)procs, (unsigned long long)best.grid.q[0], (unsigned long long)best.grid.q[1],
                    (unsigned long long)best.grid.q[2], gap < 1e-9 ? 1 : 0,
                    std::fabs(grid.fit_from_norms() - want_fit) < 1e-10 ? 1 : 0,
                    st.tree_macs == tp::tree_cost(tree, s).total_macs ? 1 : 0, (unsigned long long)shipped,
                    (unsigned long long)best.report.total);
      }
      try {
        tp::GridHooi bad(t, s, tree, tp::uniform_scheme(tree, tp::Grid{{8, 1, 1}}), std::vector<int>(8, 0));
      } catch (const tp::Error& e) {
        std::printf("error %d\n", static_cast<int>(e.code()));  // q_0 = 8 > K_0 = 5: invalid_grid
      }
      return 0;
    }
  } catch (const tp::Error& e) {
    std::printf("tuckerplan::Error %d: %s\n", static_cast<int>(e.code()), e.what());
    return 1;
  }
  return 2;
}
