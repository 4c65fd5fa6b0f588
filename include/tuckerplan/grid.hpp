// tuckerplan (B200 engine) : processor grids — drop-in for reference grid.hpp:23-125.
#pragma once

#include <vector>

#include "problem.hpp"

namespace tuckerplan {

struct Grid {
  std::vector<u64> q;
  int n_modes() const { return static_cast<int>(q.size()); }
  bool operator==(const Grid& o) const { return q == o.q; }
};

inline u64 grid_procs(const Grid& g) {
  u64 p = 1;
  for (u64 v : g.q) p = checked_mul(p, v);
  return p;
}

inline void validate_grid(const Grid& g, const ProblemSpec& s, u64 procs) {
  if (g.n_modes() != s.n_modes()) fail(Errc::invalid_grid, "grid and spec mode counts differ");
  detail::check(tp_validate_grid(s.n_modes(), s.L.data(), s.K.data(), g.q.data(), procs));
}

inline u64 grid_count(u64 procs, int n_modes) {
  u64 out = 0;
  detail::check(tp_grid_count(procs, n_modes, &out));
  return out;
}

inline std::vector<Grid> enumerate_grids(u64 procs, const ProblemSpec& s) {
  if (s.K.size() != s.L.size()) fail(Errc::bad_dims, "spec needs matching non-empty L and K");
  const int n = s.n_modes();
  std::size_t count = 0;
  std::vector<u64> flat(static_cast<std::size_t>(64) * (n > 0 ? n : 1));
  int status = tp_enumerate_grids(n, s.L.data(), s.K.data(), procs, 64, flat.data(), &count);
  if (status == TP_ERR_CAPACITY) {
    flat.resize(count * n);
    status = tp_enumerate_grids(n, s.L.data(), s.K.data(), procs, count, flat.data(), &count);
  }
  detail::check(status);
  std::vector<Grid> out(count);
  for (std::size_t i = 0; i < count; ++i) out[i].q.assign(flat.begin() + i * n, flat.begin() + (i + 1) * n);
  return out;
}

inline std::vector<u64> block_bounds(u64 len, u64 parts) {
  std::vector<u64> cuts(parts + 1);
  detail::check(tp_block_bounds(len, parts, cuts.data()));
  return cuts;
}

inline u64 block_of(u64 c, u64 len, u64 parts) {
  u64 out = 0;
  detail::check(tp_block_of(c, len, parts, &out));
  return out;
}

}  // namespace tuckerplan
