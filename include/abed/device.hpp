// abed/device.hpp -- glue between the host-side abed:: value types and the C ABI
// of libabed_b200.so.  Status codes become the reference's exception types
// (std::invalid_argument / std::out_of_range / std::runtime_error); a missing
// B200 is a runtime_error -- there is no host fallback.
#pragma once

#include <cstddef>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../abed_b200.h"
#include "tensor.hpp"

namespace abed::device {

inline void check(int status) {
  if (status == ABED_OK) return;
  const std::string msg = abed_last_error();
  if (status == ABED_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (status == ABED_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

/// Owning device allocation (RAII).
class Buffer {
 public:
  Buffer() = default;
  explicit Buffer(std::size_t bytes) : bytes_(bytes) { check(abed_malloc(&p_, bytes ? bytes : 16)); }
  ~Buffer() {
    if (p_) abed_free(p_);
  }
  Buffer(Buffer&& o) noexcept : p_(o.p_), bytes_(o.bytes_) { o.p_ = nullptr; }
  Buffer& operator=(Buffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(bytes_, o.bytes_);
    return *this;
  }
  Buffer(const Buffer&) = delete;
  Buffer& operator=(const Buffer&) = delete;
  template <typename T = void>
  T* get() const { return static_cast<T*>(p_); }
  std::size_t size() const { return bytes_; }

 private:
  void* p_ = nullptr;
  std::size_t bytes_ = 0;
};

inline Buffer upload(const void* src, std::size_t bytes) {
  Buffer b(bytes);
  if (bytes) check(abed_memcpy_h2d(b.get(), src, bytes));
  return b;
}
inline Buffer upload(const Tensor4D& t) { return upload(t.raw(), t.byte_size()); }
inline void download(const Buffer& b, void* dst, std::size_t bytes) {
  if (bytes) check(abed_memcpy_d2h(dst, b.get(), bytes));
}
inline Tensor4D download(const Buffer& b, Dims4 d, ElemKind k) {
  Tensor4D t(d, k);
  download(b, t.raw(), t.byte_size());
  return t;
}

inline abed_layer_shape c_shape(const LayerShape& s) {
  return abed_layer_shape{s.n, s.c, s.h, s.w, s.k, s.r, s.s, s.stride_h, s.stride_w, s.pad_h, s.pad_w, s.p, s.q};
}
inline abed_dims4 c_dims(Dims4 d) { return abed_dims4{d.d0, d.d1, d.d2, d.d3}; }

}  // namespace abed::device
