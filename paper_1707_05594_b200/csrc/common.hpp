// Shared host-side plumbing: status codes, the thread-local error slot, and
// exact 64-bit arithmetic for planner quantities.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "tuckerplan_b200.h"

namespace tpb {

using u64 = std::uint64_t;

// Carries a C-ABI status code through host code; converted to an int return
// (plus tp_last_error) at the extern "C" boundary.  Codes 1..13 mirror the
// reference's Errc ordinals + 1 (reference errors.hpp:16-30).
struct Failure : std::runtime_error {
  int status;
  int mode;
  Failure(int status_, const std::string& what, int mode_ = -1)
      : std::runtime_error(what), status(status_), mode(mode_) {}
};

[[noreturn]] inline void raise(int status, const std::string& what, int mode = -1) {
  throw Failure(status, what, mode);
}

void set_last_error(int status, const std::string& what, int mode);

// Runs `body`, mapping Failure/any exception to a status code.
template <class Body>
int guarded(Body&& body) noexcept {
  try {
    body();
    return TP_OK;
  } catch (const Failure& f) {
    set_last_error(f.status, f.what(), f.mode);
    return f.status;
  } catch (const std::bad_alloc&) {
    set_last_error(TP_ERR_TOO_LARGE, "host allocation failed", -1);
    return TP_ERR_TOO_LARGE;
  } catch (const std::exception& e) {
    set_last_error(TP_ERR_INTERNAL, e.what(), -1);
    return TP_ERR_INTERNAL;
  }
}

// --- exact u64 arithmetic (reference checked.hpp:18-57 semantics) -----------
constexpr u64 kSat = ~u64{0};

inline u64 mul_or_throw(u64 a, u64 b) {
  const unsigned __int128 w = static_cast<unsigned __int128>(a) * b;
  if (w > kSat) raise(TP_ERR_OVERFLOW, "64-bit overflow in product");
  return static_cast<u64>(w);
}
inline u64 add_or_throw(u64 a, u64 b) {
  const u64 r = a + b;
  if (r < a) raise(TP_ERR_OVERFLOW, "64-bit overflow in sum");
  return r;
}
inline u64 mul_sat(u64 a, u64 b) {
  const unsigned __int128 w = static_cast<unsigned __int128>(a) * b;
  return w > kSat ? kSat : static_cast<u64>(w);
}
inline u64 add_sat(u64 a, u64 b) {
  const u64 r = a + b;
  return r < a ? kSat : r;
}
// a * num / den, exact at the tensor level.
inline u64 scale_exact(u64 a, u64 num, u64 den) {
  unsigned __int128 w = static_cast<unsigned __int128>(a) * num;
  if (w % den != 0) raise(TP_ERR_OVERFLOW, "inexact division in cardinality update");
  w /= den;
  if (w > kSat) raise(TP_ERR_OVERFLOW, "64-bit overflow in cardinality update");
  return static_cast<u64>(w);
}

}  // namespace tpb
