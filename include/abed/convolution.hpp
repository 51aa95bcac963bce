// abed/convolution.hpp -- drop-in for the reference's convolution.hpp.
//
//   conv_direct (:237) / detail::conv_fast_i8 (:224)  -> tcgen05 implicit GEMM (abed_conv_i8)
//   conv_direct_f32 (:245)                            -> abed_conv_f32 (reference f32 order)
//   epilog (:353)                                     -> abed_epilog
//   im2col (:252), filters_as_matrix (:313)           -> host data rearrangement (unchanged)
//   conv_via_gemm (:323)                              -> same result as conv_direct (tcgen05)
// The reference's generic scalar `gemm` (:295, an oracle-side utility) is not
// part of the drop-in; see DESIGN.md "Out of scope".
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "device.hpp"
#include "tensor.hpp"

namespace abed {

inline constexpr std::int64_t kMaxCrsForI32 = 65536;

struct Matrix {
  std::int64_t rows = 0, cols = 0;
  ElemKind kind = ElemKind::I8;
  std::vector<std::byte> data;
  Matrix() = default;
  Matrix(std::int64_t r, std::int64_t c, ElemKind k) : rows(r), cols(c), kind(k) {
    if (r < 1 || c < 1) throw std::invalid_argument("Matrix: extents must be >= 1");
    data.resize(static_cast<std::size_t>(r * c) * elem_size(k));
  }
  std::int64_t count() const { return rows * cols; }
  template <typename T>
  std::span<T> view() {
    if (kind_of<std::remove_const_t<T>>() != kind) throw std::invalid_argument("Matrix: element access with mismatched kind");
    return {reinterpret_cast<T*>(data.data()), static_cast<std::size_t>(count())};
  }
  template <typename T>
  std::span<const T> view() const {
    if (kind_of<std::remove_const_t<T>>() != kind) throw std::invalid_argument("Matrix: element access with mismatched kind");
    return {reinterpret_cast<const T*>(data.data()), static_cast<std::size_t>(count())};
  }
  template <typename T>
  T& at(std::int64_t i, std::int64_t j) { return view<T>()[static_cast<std::size_t>(i * cols + j)]; }
  template <typename T>
  T at(std::int64_t i, std::int64_t j) const { return view<const T>()[static_cast<std::size_t>(i * cols + j)]; }
  bool operator==(const Matrix&) const = default;
};

namespace detail {

inline void check_conv_args(const Tensor4D& x, const Tensor4D& f, const LayerShape& ls, ElemKind kx, ElemKind kf) {
  if (x.kind() != kx || x.dims() != ls.input_dims()) throw std::invalid_argument("conv: input tensor does not match shape");
  if (f.kind() != kf || f.dims() != ls.filter_dims()) throw std::invalid_argument("conv: filter tensor does not match shape");
}

/// int8 convolution on the tcgen05 implicit-GEMM path; bit-identical to conv_direct.
inline Tensor4D conv_fast_i8(const Tensor4D& x, const Tensor4D& f, const LayerShape& ls) {
  check_conv_args(x, f, ls, ElemKind::I8, ElemKind::I8);
  const device::Buffer dx = device::upload(x), df = device::upload(f);
  device::Buffer out(static_cast<std::size_t>(ls.nkpq()) * 4);
  const abed_layer_shape s = device::c_shape(ls);
  device::check(abed_conv_i8(dx.get<int8_t>(), df.get<int8_t>(), &s, out.get<int32_t>(), nullptr));
  return device::download(out, ls.output_dims(), ElemKind::I32);
}

}  // namespace detail

inline Tensor4D conv_direct(const Tensor4D& x, const Tensor4D& f, const LayerShape& ls) {
  if (ls.crs() > kMaxCrsForI32)
    throw std::invalid_argument("conv_direct: CRS > 65536 exceeds the int32 accumulator plan");
  return detail::conv_fast_i8(x, f, ls);
}

inline Tensor4D conv_direct_f32(const Tensor4D& x, const Tensor4D& f, const LayerShape& ls) {
  detail::check_conv_args(x, f, ls, ElemKind::F32, ElemKind::F32);
  const device::Buffer dx = device::upload(x), df = device::upload(f);
  device::Buffer out(static_cast<std::size_t>(ls.nkpq()) * 4);
  const abed_layer_shape s = device::c_shape(ls);
  device::check(abed_conv_f32(dx.get<float>(), df.get<float>(), &s, out.get<float>(), nullptr));
  return device::download(out, ls.output_dims(), ElemKind::F32);
}

/// (C*R*S) x (N*P*Q) patch matrix; column (n,p,q) is the flattened window.
inline Matrix im2col(const Tensor4D& x, const LayerShape& ls) {
  if (x.kind() != ElemKind::I8 || x.dims() != ls.input_dims())
    throw std::invalid_argument("im2col: input tensor does not match shape");
  Matrix m(ls.crs(), ls.npq(), ElemKind::I8);
  auto mv = m.view<std::int8_t>();
  const std::int64_t npq = ls.npq();
  for (std::int64_t n = 0; n < ls.n; ++n)
    for (std::int64_t p = 0; p < ls.p; ++p)
      for (std::int64_t q = 0; q < ls.q; ++q) {
        const std::int64_t col = (n * ls.p + p) * ls.q + q;
        for_each_patch_element(x, ls, n, p, q, [&](std::int64_t c, std::int64_t r, std::int64_t s, std::int8_t v) {
          mv[static_cast<std::size_t>(((c * ls.r + r) * ls.s + s) * npq + col)] = v;
        });
      }
  return m;
}

inline Matrix filters_as_matrix(const Tensor4D& f) {
  if (f.kind() != ElemKind::I8) throw std::invalid_argument("filters_as_matrix: expected i8 filters");
  Matrix m(f.dims().d0, f.dims().d1 * f.dims().d2 * f.dims().d3, ElemKind::I8);
  std::memcpy(m.data.data(), f.raw(), f.byte_size());
  return m;
}

inline Tensor4D conv_via_gemm(const Tensor4D& x, const Tensor4D& f, const LayerShape& ls) {
  detail::check_conv_args(x, f, ls, ElemKind::I8, ElemKind::I8);
  if (ls.crs() > kMaxCrsForI32)
    throw std::invalid_argument("conv_via_gemm: CRS > 65536 exceeds the int32 accumulator plan");
  return detail::conv_fast_i8(x, f, ls);  // the device conv *is* an implicit GEMM
}

enum class Activation { ReLU, Identity };

struct EpilogParams {
  float scale = 1.0f;
  std::vector<float> bias;
  Activation activation = Activation::ReLU;
  ElemKind output_kind = ElemKind::I8;
};

namespace detail {
/// EpilogParams with the bias in device memory, for the C ABI.
struct DeviceEpilog {
  device::Buffer bias;
  abed_epilog_params c{};
  explicit DeviceEpilog(const EpilogParams& p) {
    bias = device::upload(p.bias.data(), p.bias.size() * sizeof(float));
    c = abed_epilog_params{p.scale, p.bias.empty() ? nullptr : bias.get<float>(), static_cast<int64_t>(p.bias.size()),
                           p.activation == Activation::ReLU ? ABED_RELU : ABED_IDENTITY,
                           static_cast<int32_t>(p.output_kind)};
  }
};
}  // namespace detail

inline Tensor4D epilog(const Tensor4D& convout, const EpilogParams& params) {
  if (convout.kind() != ElemKind::I32) throw std::invalid_argument("epilog: convout must be i32");
  const Dims4 d = convout.dims();
  if (static_cast<std::int64_t>(params.bias.size()) != d.d1)
    throw std::invalid_argument("epilog: bias length must equal the channel count");
  if (params.output_kind != ElemKind::I8 && params.output_kind != ElemKind::F32)
    throw std::invalid_argument("epilog: output kind must be i8 or f32");
  const detail::DeviceEpilog ep(params);
  const device::Buffer in = device::upload(convout);
  device::Buffer out(static_cast<std::size_t>(d.count()) * elem_size(params.output_kind));
  device::check(abed_epilog(in.get<int32_t>(), device::c_dims(d), &ep.c, out.get(), nullptr));
  return device::download(out, d, params.output_kind);
}

}  // namespace abed
