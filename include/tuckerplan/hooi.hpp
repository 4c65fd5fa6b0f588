// tuckerplan (B200 engine) : alternating factor updates — drop-in for reference hooi.hpp:32-245.
// Same names, argument meaning and error behaviour; the work happens in libtuckerplan_b200.so (sm_100a).
// For many sweeps on one tensor prefer `DeviceHooi`, which keeps the tensor and the factors resident in HBM —
// the by-value `hooi_sweep` re-uploads the tensor on every call, exactly as its signature implies.
#pragma once

#include <algorithm>
#include <vector>

#include "problem.hpp"
#include "ttm.hpp"
#include "ttm_tree.hpp"

namespace tuckerplan {

inline constexpr std::size_t kMaxGramRows = TP_MAX_GRAM_ROWS;
inline constexpr double kDegenerateGap = 1e-10;

struct TruncatedBasis {
  Matrix vectors;  // rows x k, orthonormal, descending eigenvalues
  bool degenerate = false;
};

template <class M>
TruncatedBasis leading_left_factors(const M& m, int k, DeviceContext& dev = DeviceContext::instance()) {
  Matrix scratch;
  const Matrix& mm = detail::as_matrix(m, scratch);
  if (mm.rows() == 0 || mm.cols() == 0) fail(Errc::shape_mismatch, "empty matrix");
  if (mm.rows() > kMaxGramRows) fail(Errc::too_large, "unfolding has too many rows for the Gram route");
  if (k < 1 || static_cast<std::size_t>(k) > mm.rows()) fail(Errc::bad_argument, "need 1 <= k <= rows");
  TruncatedBasis basis;
  basis.vectors = Matrix(mm.rows(), static_cast<std::size_t>(k));
  int degenerate = 0;
  detail::check(tp_leading_left_factors(dev.get(), mm.data(), mm.rows(), mm.cols(), k, basis.vectors.data(),
                                        &degenerate));
  basis.degenerate = degenerate != 0;
  return basis;
}

struct Decomposition {
  DenseTensor core;             // extents K
  std::vector<Matrix> factors;  // factors[n] is L_n x K_n
};

struct SweepStats {
  u64 tree_macs = 0;
  u64 core_macs = 0;
  int peak_live = 0;
  bool degenerate = false;
};

enum class SweepKind { jacobi, gauss_seidel };

namespace detail {
inline void check_engine_shapes(const DenseTensor& t, const ProblemSpec& s) {
  if (t.n_modes() != s.n_modes()) fail(Errc::shape_mismatch, "tensor and spec mode counts differ");
  for (int m = 0; m < s.n_modes(); ++m)
    if (t.dims[m] != s.L[m]) fail(Errc::shape_mismatch, "tensor extent differs from L", m);
}
inline DenseTensor core_from_factors(const DenseTensor& t, const std::vector<Matrix>& factors, u64* macs = nullptr) {
  DenseTensor z = t;
  for (std::size_t n = 0; n < factors.size(); ++n) z = ttm(z, factors[n].transpose(), static_cast<int>(n), macs);
  return z;
}
}  // namespace detail

inline Decomposition random_decomposition(const DenseTensor& t, const ProblemSpec& s, std::uint64_t seed) {
  validate_spec(s);
  detail::check_engine_shapes(t, s);
  Decomposition d;
  std::vector<double*> ptrs;
  for (int n = 0; n < s.n_modes(); ++n) {
    d.factors.emplace_back(s.L[n], s.K[n]);
    ptrs.push_back(d.factors.back().data());
  }
  for (int n = 0; n < s.n_modes(); ++n) ptrs[n] = d.factors[n].data();
  detail::check(tp_random_orthonormal_factors(s.n_modes(), s.L.data(), s.K.data(), seed, ptrs.data()));
  d.core = detail::core_from_factors(t, d.factors);
  return d;
}

inline Decomposition hooi_sweep(const DenseTensor& t, const ProblemSpec& s, const Decomposition& d,
                                const TtmTree& tree, SweepKind kind, SweepStats* stats = nullptr,
                                DeviceContext& dev = DeviceContext::instance()) {
  detail::check_engine_shapes(t, s);
  validate_tree(tree, s);
  if (d.factors.size() != static_cast<std::size_t>(s.n_modes()))
    fail(Errc::shape_mismatch, "factor count differs from mode count");
  if (stats) *stats = SweepStats{};
  const detail::FlatTree f = detail::flatten(tree);
  Decomposition out;
  std::vector<const double*> in_ptrs;
  std::vector<double*> out_ptrs;
  std::vector<std::size_t> core_dims;
  for (int n = 0; n < s.n_modes(); ++n) {
    if (d.factors[n].rows() != s.L[n] || d.factors[n].cols() != s.K[n])
      fail(Errc::shape_mismatch, "factor shape differs from L x K", n);
    out.factors.emplace_back(s.L[n], s.K[n]);
    core_dims.push_back(s.K[n]);
  }
  for (int n = 0; n < s.n_modes(); ++n) {
    in_ptrs.push_back(d.factors[n].data());
    out_ptrs.push_back(out.factors[n].data());
  }
  out.core = zeros(core_dims);
  tp_sweep_stats st{};
  detail::check(tp_hooi_sweep_host(dev.get(), s.n_modes(), t.dims.data(), t.data.data(), s.K.data(), in_ptrs.data(),
                                   f.size(), f.kind.data(), f.mode.data(), f.parent.data(),
                                   kind == SweepKind::jacobi ? TP_SWEEP_JACOBI : TP_SWEEP_GAUSS_SEIDEL,
                                   out_ptrs.data(), out.core.data.data(), &st));
  if (stats) *stats = SweepStats{st.tree_macs, st.core_macs, st.peak_live, st.degenerate != 0};
  return out;
}

inline double reconstruction_error(const DenseTensor& t, const Decomposition& d,
                                   DeviceContext& dev = DeviceContext::instance()) {
  if (t.dims.empty()) fail(Errc::zero_tensor, "relative error undefined at zero");
  detail::TensorHandle in(dev.get(), t);
  const bool shapes_ok = d.core.n_modes() == t.n_modes() && d.factors.size() == t.dims.size();
  std::vector<const double*> ptrs;
  bool factors_ok = shapes_ok;
  for (std::size_t n = 0; shapes_ok && n < d.factors.size(); ++n) {
    factors_ok = factors_ok && d.factors[n].rows() == t.dims[n] && d.factors[n].cols() == d.core.dims[n];
    ptrs.push_back(d.factors[n].data());
  }
  double out = 0.0;
  // the reference evaluates the norm first (zero_tensor), then fails on the shape (hooi.hpp:233-238)
  detail::check(tp_reconstruction_error(dev.get(), in.t, factors_ok ? d.core.dims.data() : nullptr,
                                        factors_ok ? d.core.data.data() : nullptr,
                                        factors_ok ? ptrs.data() : nullptr, &out));
  return out;
}

// Sequentially truncated HOSVD start: for each mode in turn the leading K_n left singular vectors of the current
// unfolding (selected and signed as leading_left_factors does), the tensor truncated along that mode before the next.
// Not in the reference (SPEC.md:17 leaves starts other than random_decomposition out of scope); it is what HOOI is
// usually started from and costs about one sweep.  `degenerate` (optional) receives the OR of the
// leaves' gap flags.
inline Decomposition sthosvd(const DenseTensor& t, const ProblemSpec& s, bool* degenerate = nullptr,
                             DeviceContext& dev = DeviceContext::instance()) {
  validate_spec(s);
  detail::check_engine_shapes(t, s);
  detail::TensorHandle handle(dev.get(), t);
  Decomposition d;
  std::vector<std::size_t> core_dims;
  std::vector<double*> ptrs;
  for (int n = 0; n < s.n_modes(); ++n) {
    d.factors.emplace_back(s.L[n], s.K[n]);
    core_dims.push_back(s.K[n]);
  }
  for (Matrix& f : d.factors) ptrs.push_back(f.data());
  d.core = zeros(core_dims);
  int flag = 0;
  detail::check(tp_sthosvd(dev.get(), handle.t, s.K.data(), nullptr, ptrs.data(), d.core.data.data(), &flag, nullptr));
  if (degenerate) *degenerate = flag != 0;
  return d;
}

// Resident form of the sweep driver: tensor, factors, intermediates and the launch schedule stay in HBM.
class DeviceHooi {
 public:
  DeviceHooi(const DenseTensor& t, const ProblemSpec& s, const TtmTree& tree, SweepKind kind,
             DeviceContext& dev = DeviceContext::instance())
      : dev_(dev), spec_(s), tensor_(dev.get(), t) {
    detail::check_engine_shapes(t, s);
    validate_tree(tree, s);
    const detail::FlatTree f = detail::flatten(tree);
    detail::check(tp_plan_create(dev.get(), s.n_modes(), s.L.data(), s.K.data(), f.size(), f.kind.data(),
                                 f.mode.data(), f.parent.data(),
                                 kind == SweepKind::jacobi ? TP_SWEEP_JACOBI : TP_SWEEP_GAUSS_SEIDEL, &plan_));
  }
  ~DeviceHooi() { if (plan_) tp_plan_destroy(dev_.get(), plan_); }
  DeviceHooi(const DeviceHooi&) = delete;
  DeviceHooi& operator=(const DeviceHooi&) = delete;

  void set_factors(const std::vector<Matrix>& factors) {
    if (factors.size() != static_cast<std::size_t>(spec_.n_modes()))
      fail(Errc::shape_mismatch, "factor count differs from mode count");
    std::vector<const double*> ptrs;
    for (const Matrix& f : factors) ptrs.push_back(f.data());
    detail::check(tp_plan_set_factors(dev_.get(), plan_, ptrs.data()));
  }
  SweepStats sweep() {
    tp_sweep_stats st{};
    detail::check(tp_plan_sweep(dev_.get(), plan_, tensor_.t, &st));
    return SweepStats{st.tree_macs, st.core_macs, st.peak_live, st.degenerate != 0};
  }
  Decomposition decomposition() {
    Decomposition d;
    std::vector<std::size_t> core_dims;
    std::vector<double*> ptrs;
    for (int n = 0; n < spec_.n_modes(); ++n) {
      d.factors.emplace_back(spec_.L[n], spec_.K[n]);
      core_dims.push_back(spec_.K[n]);
    }
    for (Matrix& f : d.factors) ptrs.push_back(f.data());
    detail::check(tp_plan_get_factors(dev_.get(), plan_, ptrs.data()));
    d.core = zeros(core_dims);
    detail::check(tp_plan_get_core(dev_.get(), plan_, d.core.data.data()));
    return d;
  }
  double reconstruction_error() {
    double out = 0.0;
    detail::check(tp_plan_reconstruction_error(dev_.get(), plan_, tensor_.t, &out));
    return out;
  }
  tp_sweep_timing last_timing() {
    tp_sweep_timing tm{};
    detail::check(tp_plan_last_timing(dev_.get(), plan_, &tm));
    return tm;
  }

 private:
  DeviceContext& dev_;
  ProblemSpec spec_;
  detail::TensorHandle tensor_;
  tp_plan* plan_ = nullptr;
};

// Jacobi sweeps on a Cartesian processor grid: rank p of `scheme` (row-major block order, simulate.hpp:69-73) runs on
// CUDA device devices[p] of this box; the same device may be named several times.  A static grid is
// uniform_scheme(tree, grid) (simulate.hpp:50-57); optimal_dynamic_scheme(...).scheme gives per-node grids with
// regrids.  What the reference only simulates (simulate_distribution) is executed here; last_volumes() returns the
// elements actually shipped per node, to be compared with the ledger's model columns.
class GridHooi {
 public:
  GridHooi(const DenseTensor& t, const ProblemSpec& s, const TtmTree& tree, const DynamicGridScheme& scheme,
           const std::vector<int>& devices, bool use_nccl = false)
      : spec_(s), n_nodes_(static_cast<int>(tree.nodes.size())) {
    detail::check_engine_shapes(t, s);
    validate_tree(tree, s);
    const detail::FlatTree f = detail::flatten(tree);
    std::vector<u64> node_grids(static_cast<std::size_t>(f.size()) * s.n_modes(), 0);
    for (int id = 0; id < f.size(); ++id) {
      if (!tree.is_internal(id)) continue;
      const auto it = scheme.node_grids.find(id);
      if (it == scheme.node_grids.end()) fail(Errc::missing_assignment, "scheme has no grid for node " + std::to_string(id));
      if (it->second.n_modes() != s.n_modes()) fail(Errc::invalid_grid, "grid and spec mode counts differ");
      std::copy(it->second.q.begin(), it->second.q.end(), node_grids.begin() + static_cast<std::size_t>(id) * s.n_modes());
    }
    if (scheme.root.n_modes() != s.n_modes()) fail(Errc::invalid_grid, "grid and spec mode counts differ");
    detail::check(tp_grid_create(static_cast<int>(devices.size()), devices.data(), s.n_modes(), s.L.data(), s.K.data(),
                                 f.size(), f.kind.data(), f.mode.data(), f.parent.data(), scheme.root.q.data(),
                                 node_grids.data(), use_nccl ? static_cast<unsigned>(TP_GRID_NCCL) : 0u, &grid_));
    const int status = tp_grid_set_tensor(grid_, t.data.data());
    if (status != TP_OK) {
      tp_grid_destroy(grid_);
      grid_ = nullptr;
      detail::check(status);
    }
  }
  ~GridHooi() { if (grid_) tp_grid_destroy(grid_); }
  GridHooi(const GridHooi&) = delete;
  GridHooi& operator=(const GridHooi&) = delete;

  void set_factors(const std::vector<Matrix>& factors) {
    if (factors.size() != static_cast<std::size_t>(spec_.n_modes()))
      fail(Errc::shape_mismatch, "factor count differs from mode count");
    std::vector<const double*> ptrs;
    for (const Matrix& f : factors) ptrs.push_back(f.data());
    detail::check(tp_grid_set_factors(grid_, ptrs.data()));
  }
  SweepStats sweep() {
    tp_sweep_stats st{};
    detail::check(tp_grid_sweep(grid_, &st));
    return SweepStats{st.tree_macs, st.core_macs, st.peak_live, st.degenerate != 0};
  }
  Decomposition decomposition() {
    Decomposition d;
    std::vector<std::size_t> core_dims;
    std::vector<double*> ptrs;
    for (int n = 0; n < spec_.n_modes(); ++n) {
      d.factors.emplace_back(spec_.L[n], spec_.K[n]);
      core_dims.push_back(spec_.K[n]);
    }
    for (Matrix& f : d.factors) ptrs.push_back(f.data());
    detail::check(tp_grid_get_factors(grid_, ptrs.data()));
    d.core = zeros(core_dims);
    detail::check(tp_grid_get_core(grid_, d.core.data.data()));
    return d;
  }
  // sqrt(||T||^2 - ||G||^2) / ||T||: the relative error of a decomposition with orthonormal factors and their core
  double fit_from_norms() {
    double out = 0.0;
    detail::check(tp_grid_fit_from_norms(grid_, &out));
    return out;
  }
  struct Volumes {
    std::vector<u64> ttm, regrid;  // per tree node, elements shipped by all ranks in the last sweep
  };
  Volumes last_volumes() const {
    Volumes v{std::vector<u64>(n_nodes_, 0), std::vector<u64>(n_nodes_, 0)};
    detail::check(tp_grid_last_volumes(grid_, n_nodes_, v.ttm.data(), v.regrid.data()));
    return v;
  }
  float last_total_ms() const {
    float ms = 0.f;
    detail::check(tp_grid_last_timing(grid_, &ms, 0, nullptr, nullptr));
    return ms;
  }

 private:
  ProblemSpec spec_;
  int n_nodes_ = 0;
  tp_grid* grid_ = nullptr;
};

}  // namespace tuckerplan
