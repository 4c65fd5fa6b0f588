// tuckerplan (B200 engine) : mode products and unfoldings — drop-in for reference ttm.hpp:43-96.
// `ttm` runs on the GPU (strided DMMA kernel, no unfolding is ever formed); `unfold` / `fold` are kept for API
// parity as plain host index maps — the engine itself never calls them.
#pragma once

#include <cstdint>
#include <memory>

#include "checked.hpp"
#include "dense_tensor.hpp"
#include "matrix.hpp"

namespace tuckerplan {

// One CUDA device + stream (tp_ctx).  Functions taking host values use a process-wide default context on device 0
// unless told otherwise; a context is not thread-safe (use one per host thread).
class DeviceContext {
 public:
  explicit DeviceContext(int device = 0) { detail::check(tp_ctx_create(device, &ctx_)); }
  ~DeviceContext() { if (ctx_) tp_ctx_destroy(ctx_); }
  DeviceContext(const DeviceContext&) = delete;
  DeviceContext& operator=(const DeviceContext&) = delete;
  tp_ctx* get() const { return ctx_; }
  static DeviceContext& instance() {
    static thread_local DeviceContext ctx(0);
    return ctx;
  }

 private:
  tp_ctx* ctx_ = nullptr;
};

namespace detail {
inline void mode_extents(const DenseTensor& t, int mode, std::size_t& outer, std::size_t& inner) {
  if (mode < 0 || mode >= t.n_modes()) fail(Errc::bad_mode, "mode out of range", mode);
  outer = inner = 1;
  for (int m = 0; m < mode; ++m) outer *= t.dims[m];
  for (int m = mode + 1; m < t.n_modes(); ++m) inner *= t.dims[m];
}
struct TensorHandle {  // RAII for tp_tensor
  tp_ctx* ctx = nullptr;
  tp_tensor* t = nullptr;
  TensorHandle() = default;
  TensorHandle(tp_ctx* c, const DenseTensor& host) : ctx(c) {
    check(tp_tensor_upload(ctx, host.n_modes(), host.dims.data(), host.data.data(), &t));
  }
  ~TensorHandle() { if (t) tp_tensor_free(ctx, t); }
  TensorHandle(const TensorHandle&) = delete;
  TensorHandle& operator=(const TensorHandle&) = delete;
};
}  // namespace detail

// Column a * inner + b of the result is fibre (a, :, b) (reference ttm.hpp:4-8, 43-53).
inline Matrix unfold(const DenseTensor& t, int mode) {
  std::size_t outer, inner;
  detail::mode_extents(t, mode, outer, inner);
  const std::size_t len = t.dims[mode];
  Matrix m(len, outer * inner);
  for (std::size_t a = 0; a < outer; ++a)
    for (std::size_t i = 0; i < len; ++i)
      for (std::size_t b = 0; b < inner; ++b) m(i, a * inner + b) = t.data[(a * len + i) * inner + b];
  return m;
}

template <class M>
DenseTensor fold(const M& m, std::vector<std::size_t> dims, int mode) {
  DenseTensor t = zeros(std::move(dims));
  std::size_t outer, inner;
  detail::mode_extents(t, mode, outer, inner);
  const std::size_t len = t.dims[mode];
  if (static_cast<std::size_t>(m.rows()) != len || static_cast<std::size_t>(m.cols()) != outer * inner)
    fail(Errc::shape_mismatch, "matrix does not match the unfolding shape");
  for (std::size_t a = 0; a < outer; ++a)
    for (std::size_t i = 0; i < len; ++i)
      for (std::size_t b = 0; b < inner; ++b) t.data[(a * len + i) * inner + b] = m(i, a * inner + b);
  return t;
}

// t x_mode m with m of shape (new_len x dims[mode]); *macs is ACCUMULATED with new_len * t.size().
template <class M>
DenseTensor ttm(const DenseTensor& t, const M& m, int mode, u64* macs = nullptr,
                DeviceContext& dev = DeviceContext::instance()) {
  Matrix scratch;
  const Matrix& mm = detail::as_matrix(m, scratch);
  std::size_t outer, inner;
  detail::mode_extents(t, mode, outer, inner);
  if (mm.cols() != t.dims[mode]) fail(Errc::shape_mismatch, "matrix columns must match the mode extent");
  if (mm.rows() == 0) fail(Errc::shape_mismatch, "empty matrix");
  detail::TensorHandle in(dev.get(), t);
  detail::TensorHandle out;
  out.ctx = dev.get();
  detail::check(tp_ttm(dev.get(), in.t, mm.data(), mm.rows(), mm.cols(), mode, macs, &out.t));
  DenseTensor z;
  z.dims = t.dims;
  z.dims[mode] = mm.rows();
  z.data.resize(z.size());
  detail::check(tp_tensor_download(dev.get(), out.t, z.data.data()));
  return z;
}

}  // namespace tuckerplan
