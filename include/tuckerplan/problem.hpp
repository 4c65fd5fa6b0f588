// tuckerplan (B200 engine) : problem specification — drop-in for reference problem.hpp:22-86.
#pragma once

#include <vector>

#include "checked.hpp"
#include "mode_set.hpp"

namespace tuckerplan {

inline constexpr u64 kMaxElements = u64{1} << 62;

struct ProblemSpec {
  std::vector<u64> L;
  std::vector<u64> K;
  int n_modes() const { return static_cast<int>(L.size()); }
};

struct Ratio {
  u64 num;
  u64 den;
};

inline void validate_spec(const ProblemSpec& s) {
  if (s.K.size() != s.L.size()) fail(Errc::bad_dims, "spec needs matching non-empty L and K");
  detail::check(tp_validate_spec(s.n_modes(), s.L.data(), s.K.data()));
}
inline u64 cost_factor(const ProblemSpec& s, int mode) {
  if (mode < 0 || mode >= s.n_modes()) fail(Errc::bad_mode, "mode out of range", mode);
  return s.K[mode];
}
inline Ratio compression_factor(const ProblemSpec& s, int mode) {
  if (mode < 0 || mode >= s.n_modes()) fail(Errc::bad_mode, "mode out of range", mode);
  return Ratio{s.K[mode], s.L[mode]};
}
inline u64 partial_cardinality(const ProblemSpec& s, ModeSet done) {
  u64 out = 0;
  detail::check(tp_partial_cardinality(s.n_modes(), s.L.data(), s.K.data(), done.bits(), &out));
  return out;
}
inline u64 input_cardinality(const ProblemSpec& s) { return partial_cardinality(s, ModeSet()); }
inline u64 core_cardinality(const ProblemSpec& s) { return partial_cardinality(s, ModeSet::full(s.n_modes())); }

}  // namespace tuckerplan
