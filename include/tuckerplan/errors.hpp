// tuckerplan (B200 engine) : error reporting — drop-in for reference errors.hpp.
// Same enum names and order as the reference (errors.hpp:16-30) so that callers' `e.code() == Errc::...`
// comparisons keep compiling; the codes travel through the C ABI as ordinal + 1 (include/tuckerplan_b200.h).
#pragma once

#include <stdexcept>
#include <string>

#include "../tuckerplan_b200.h"

namespace tuckerplan {

enum class Errc {
  bad_dims, k_too_large, overflow, bad_tree, bad_mode, shape_mismatch, invalid_grid, no_valid_grid,
  missing_assignment, too_large, zero_tensor, needs_chain_tree, bad_argument,
  // not in the reference: failures of the device layer
  cuda_failure, nccl_failure, capacity, internal
};

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what, int mode = -1) : std::runtime_error(what), code_(code), mode_(mode) {}
  Errc code() const noexcept { return code_; }
  int mode() const noexcept { return mode_; }

 private:
  Errc code_;
  int mode_;
};

[[noreturn]] inline void fail(Errc code, const std::string& what, int mode = -1) { throw Error(code, what, mode); }

namespace detail {
inline Errc errc_from_status(int status) {
  if (status >= 1 && status <= 13) return static_cast<Errc>(status - 1);
  switch (status) {
    case TP_ERR_CUDA: return Errc::cuda_failure;
    case TP_ERR_NCCL: return Errc::nccl_failure;
    case TP_ERR_CAPACITY: return Errc::capacity;
    default: return Errc::internal;
  }
}
// Rethrows a C-ABI failure as the reference's exception type.
inline void check(int status) {
  if (status != TP_OK) throw Error(errc_from_status(status), tp_last_error(), tp_last_error_mode());
}
}  // namespace detail

}  // namespace tuckerplan
