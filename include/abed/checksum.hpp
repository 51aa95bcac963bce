// abed/checksum.hpp -- drop-in for the reference's checksum.hpp (the ABED schemes).
//
// Every checksum generation, plane convolution, recombination and verification
// runs on the B200 through libabed_b200.so; VerifyOutcome values (status, locus,
// lhs, rhs) are bit-identical to the reference (tests/test_gpu_parity.py).
// citations: checksum.hpp:15 Scheme, :30 VerifyOutcome, :75-206 FC, :211 fc_verify,
// :248-347 IC/FIC, :350-421 ICBatch, :429-468 planner, :474-595 float mode,
// :605-631 fused_conv_epilog.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <vector>

#include "convolution.hpp"
#include "device.hpp"
#include "tensor.hpp"

namespace abed {

enum class Scheme { FC, IC, ICBatch, FIC };

inline const char* to_string(Scheme s) {
  constexpr const char* names[] = {"fc", "ic", "icbatch", "fic"};
  return names[static_cast<int>(s)];
}

struct VerifyOutcome {
  enum class Status { Pass, Mismatch };
  Status status = Status::Pass;
  std::optional<std::array<std::int64_t, 3>> locus;
  std::int64_t lhs = 0;
  std::int64_t rhs = 0;
  double lhs_f = 0.0, rhs_f = 0.0;

  bool pass() const { return status == Status::Pass; }
  static VerifyOutcome ok() { return {}; }
  static VerifyOutcome fail(std::int64_t lhs, std::int64_t rhs, std::optional<std::array<std::int64_t, 3>> locus = std::nullopt) {
    VerifyOutcome v;
    v.status = Status::Mismatch;
    v.lhs = lhs;
    v.rhs = rhs;
    v.locus = locus;
    return v;
  }
};

namespace detail {
inline VerifyOutcome from_c(const abed_verify_outcome& o) {
  VerifyOutcome v;
  v.status = o.status ? VerifyOutcome::Status::Mismatch : VerifyOutcome::Status::Pass;
  if (o.has_locus) v.locus = std::array<std::int64_t, 3>{o.locus[0], o.locus[1], o.locus[2]};
  v.lhs = o.lhs;
  v.rhs = o.rhs;
  v.lhs_f = o.lhs_f;
  v.rhs_f = o.rhs_f;
  return v;
}
}  // namespace detail

inline int ceil_log2(std::int64_t v) {
  if (v < 1) throw std::invalid_argument("ceil_log2: argument must be >= 1");
  int bits = 0;
  for (std::uint64_t u = static_cast<std::uint64_t>(v) - 1; u; u >>= 1) ++bits;
  return bits;
}

// ------------------------------------------------------------------ FC
struct FilterChecksum {
  Tensor4D sums;  // 1 x C x R x S, i32
  std::optional<std::array<Tensor4D, 4>> decomposed;
};

inline FilterChecksum gen_filter_checksum(const Tensor4D& filters) {
  if (filters.kind() != ElemKind::I8) throw std::invalid_argument("gen_filter_checksum: expected i8 filters");
  const Dims4 d = filters.dims();
  const device::Buffer df = device::upload(filters);
  device::Buffer out(static_cast<std::size_t>(d.d1 * d.d2 * d.d3) * 4);
  device::check(abed_gen_filter_checksum(df.get<int8_t>(), device::c_dims(d), out.get<int32_t>(), nullptr));
  return FilterChecksum{device::download(out, {1, d.d1, d.d2, d.d3}, ElemKind::I32), std::nullopt};
}

/// Little-endian byte planes of an int32 (checksum.hpp:93-97).
inline std::array<std::int8_t, 4> decompose_value(std::int32_t v) {
  const auto u = static_cast<std::uint32_t>(v);
  return {static_cast<std::int8_t>(u & 0xFF), static_cast<std::int8_t>((u >> 8) & 0xFF),
          static_cast<std::int8_t>((u >> 16) & 0xFF), static_cast<std::int8_t>(u >> 24)};
}
/// Digits 0-2 as unsigned bytes, digit 3 signed (checksum.hpp:101-106).
inline std::int64_t recombine_value(const std::array<std::int8_t, 4>& d) {
  return std::int64_t{static_cast<std::uint8_t>(d[0])} + (std::int64_t{static_cast<std::uint8_t>(d[1])} << 8) +
         (std::int64_t{static_cast<std::uint8_t>(d[2])} << 16) + std::int64_t{d[3]} * 16777216;
}

inline std::array<Tensor4D, 4> decompose_checksum_filters(const FilterChecksum& fc) {
  if (fc.sums.kind() != ElemKind::I32) throw std::invalid_argument("decompose_checksum_filters: sums must be i32");
  const Dims4 d = fc.sums.dims();
  const std::int64_t n = d.count();
  const device::Buffer ds = device::upload(fc.sums);
  device::Buffer planes(static_cast<std::size_t>(4 * n));
  device::check(abed_decompose_checksum_filters(ds.get<int32_t>(), n, planes.get<int8_t>(), nullptr));
  std::vector<std::int8_t> h(static_cast<std::size_t>(4 * n));
  device::download(planes, h.data(), h.size());
  std::array<Tensor4D, 4> out{Tensor4D(d, ElemKind::I8), Tensor4D(d, ElemKind::I8), Tensor4D(d, ElemKind::I8),
                              Tensor4D(d, ElemKind::I8)};
  for (int p = 0; p < 4; ++p) std::memcpy(out[p].raw(), h.data() + p * n, static_cast<std::size_t>(n));
  return out;
}

inline FilterChecksum gen_filter_checksum_decomposed(const Tensor4D& filters) {
  FilterChecksum fc = gen_filter_checksum(filters);
  fc.decomposed = decompose_checksum_filters(fc);
  return fc;
}

inline std::array<Tensor4D, 4> conv_checksum_planes(const Tensor4D& input, const LayerShape& ls,
                                                    const std::array<Tensor4D, 4>& planes) {
  if (ls.crs() > kMaxCrsForI32) throw std::invalid_argument("conv_checksum_planes: CRS > 65536 exceeds the i32 plan");
  const Dims4 pd{1, ls.c, ls.r, ls.s};
  std::vector<std::int8_t> hp(static_cast<std::size_t>(4 * ls.crs()));
  for (int p = 0; p < 4; ++p) {
    if (planes[p].dims() != pd || planes[p].kind() != ElemKind::I8)
      throw std::invalid_argument("conv_checksum_planes: bad plane tensor");
    std::memcpy(hp.data() + p * ls.crs(), planes[p].raw(), static_cast<std::size_t>(ls.crs()));
  }
  if (input.kind() != ElemKind::I8 || input.dims() != ls.input_dims())
    throw std::invalid_argument("conv_checksum_planes: input does not match shape");
  const device::Buffer dx = device::upload(input), dp = device::upload(hp.data(), hp.size());
  device::Buffer out(static_cast<std::size_t>(4 * ls.npq()) * 4);
  const abed_layer_shape s = device::c_shape(ls);
  device::check(abed_conv_checksum_planes(dx.get<int8_t>(), &s, dp.get<int8_t>(), out.get<int32_t>(), nullptr));
  std::vector<std::int32_t> h(static_cast<std::size_t>(4 * ls.npq()));
  device::download(out, h.data(), h.size() * 4);
  std::array<Tensor4D, 4> e;
  for (int p = 0; p < 4; ++p) {
    e[p] = Tensor4D({ls.n, 1, ls.p, ls.q}, ElemKind::I32);
    std::memcpy(e[p].raw(), h.data() + p * ls.npq(), static_cast<std::size_t>(ls.npq()) * 4);
  }
  return e;
}

inline Tensor4D recombine_extra_fmaps(const std::array<Tensor4D, 4>& extra) {
  const Dims4 d = extra[0].dims();
  const std::int64_t n = d.count();
  std::vector<std::int32_t> h(static_cast<std::size_t>(4 * n));
  for (int p = 0; p < 4; ++p) {
    if (extra[p].dims() != d || extra[p].kind() != ElemKind::I32)
      throw std::invalid_argument("recombine_extra_fmaps: planes must be matching i32 tensors");
    std::memcpy(h.data() + p * n, extra[p].raw(), static_cast<std::size_t>(n) * 4);
  }
  const device::Buffer de = device::upload(h.data(), h.size() * 4);
  device::Buffer out(static_cast<std::size_t>(n) * 8);
  device::check(abed_recombine_extra_fmaps(de.get<int32_t>(), n, out.get<int64_t>(), nullptr));
  return device::download(out, d, ElemKind::I64);
}

inline Tensor4D conv_filter_checksum(const Tensor4D& input, const LayerShape& ls, const FilterChecksum& fc) {
  const device::Buffer dx = device::upload(input), ds = device::upload(fc.sums);
  device::Buffer out(static_cast<std::size_t>(ls.npq()) * 8);
  const abed_layer_shape s = device::c_shape(ls);
  device::check(abed_conv_filter_checksum(dx.get<int8_t>(), &s, ds.get<int32_t>(), out.get<int64_t>(), nullptr));
  return device::download(out, {ls.n, 1, ls.p, ls.q}, ElemKind::I64);
}

inline VerifyOutcome fc_verify(const Tensor4D& convout, const Tensor4D& extra, std::int64_t original_k = -1) {
  if (convout.kind() != ElemKind::I32) throw std::invalid_argument("fc_verify: convout must be i32");
  if (extra.kind() != ElemKind::I64) throw std::invalid_argument("fc_verify: extra fmap must be i64");
  const Dims4 d = convout.dims();
  if (extra.dims() != Dims4{d.d0, 1, d.d2, d.d3}) throw std::invalid_argument("fc_verify: extra fmap dims do not match convout");
  const device::Buffer dc = device::upload(convout), de = device::upload(extra);
  abed_verify_outcome o{};
  device::check(abed_fc_verify(dc.get<int32_t>(), device::c_dims(d), de.get<int64_t>(), original_k, &o));
  return detail::from_c(o);
}

// ------------------------------------------------------------------ IC / FIC
struct InputChecksum {
  Tensor4D sums;  // 1 x C x R x S, i32
};

inline InputChecksum gen_input_checksum(const Tensor4D& input, const LayerShape& ls) {
  if (input.kind() != ElemKind::I8 || input.dims() != ls.input_dims())
    throw std::invalid_argument("gen_input_checksum: input does not match shape");
  const device::Buffer dx = device::upload(input);
  device::Buffer out(static_cast<std::size_t>(ls.crs()) * 4);
  const abed_layer_shape s = device::c_shape(ls);
  device::check(abed_gen_input_checksum(dx.get<int8_t>(), &s, out.get<int32_t>(), nullptr));
  return InputChecksum{device::download(out, {1, ls.c, ls.r, ls.s}, ElemKind::I32)};
}

inline std::int64_t reduce_all_i64(const Tensor4D& convout) {
  const device::Buffer dc = device::upload(convout);
  std::int64_t r = 0;
  device::check(abed_reduce_all_i64(dc.get<int32_t>(), convout.count(), &r));
  return r;
}

inline std::int64_t fic_dot(const FilterChecksum& fc, const InputChecksum& ic) {
  if (fc.sums.dims() != ic.sums.dims()) throw std::invalid_argument("fic_dot: checksum sizes do not match");
  const device::Buffer a = device::upload(fc.sums), b = device::upload(ic.sums);
  std::int64_t r = 0;
  device::check(abed_fic_dot(a.get<int32_t>(), b.get<int32_t>(), fc.sums.count(), &r));
  return r;
}

inline VerifyOutcome fic_verify(const Tensor4D& convout, std::int64_t expected) {
  const device::Buffer dc = device::upload(convout);
  abed_verify_outcome o{};
  device::check(abed_fic_verify(dc.get<int32_t>(), convout.count(), expected, &o));
  return detail::from_c(o);
}

inline std::int32_t reduce_all_wrap32(const Tensor4D& convout) {
  const device::Buffer dc = device::upload(convout);
  std::int32_t r = 0;
  device::check(abed_reduce_all_wrap32(dc.get<int32_t>(), convout.count(), &r));
  return r;
}

inline VerifyOutcome fic_verify_forced32(const Tensor4D& convout, std::int64_t expected) {
  const device::Buffer dc = device::upload(convout);
  abed_verify_outcome o{};
  device::check(abed_fic_verify_forced32(dc.get<int32_t>(), convout.count(), expected, &o));
  return detail::from_c(o);
}

inline VerifyOutcome ic_verify_k(const Tensor4D& convout, const Tensor4D& filters, const InputChecksum& ic) {
  if (convout.kind() != ElemKind::I32) throw std::invalid_argument("ic_verify_k: convout must be i32");
  if (filters.kind() != ElemKind::I8) throw std::invalid_argument("ic_verify_k: filters must be i8");
  const Dims4 fd = filters.dims();
  if (ic.sums.dims() != Dims4{1, fd.d1, fd.d2, fd.d3})
    throw std::invalid_argument("ic_verify_k: checksum size does not match filters");
  const device::Buffer dc = device::upload(convout), df = device::upload(filters), di = device::upload(ic.sums);
  abed_verify_outcome o{};
  device::check(abed_ic_verify_k(dc.get<int32_t>(), device::c_dims(convout.dims()), df.get<int8_t>(), device::c_dims(fd),
                                 di.get<int32_t>(), &o));
  return detail::from_c(o);
}

// ------------------------------------------------------------------ ICBatch
inline Tensor4D ic_batch_checksum(const Tensor4D& input) {
  if (input.kind() != ElemKind::I8) throw std::invalid_argument("ic_batch_checksum: expected i8 input");
  const Dims4 d = input.dims();
  const device::Buffer dx = device::upload(input);
  device::Buffer out(static_cast<std::size_t>(d.d1 * d.d2 * d.d3) * 4);
  device::check(abed_ic_batch_checksum(dx.get<int8_t>(), device::c_dims(d), out.get<int32_t>(), nullptr));
  return device::download(out, {1, d.d1, d.d2, d.d3}, ElemKind::I32);
}

/// Checksum image convolved as extra int8 digit images on the tcgen05 path.
inline Tensor4D conv_batch_checksum(const Tensor4D& batch, const Tensor4D& filters, const LayerShape& ls) {
  if (batch.kind() != ElemKind::I32) throw std::invalid_argument("conv_batch_checksum: batch must be i32");
  if (batch.dims() != Dims4{1, ls.c, ls.h, ls.w}) throw std::invalid_argument("conv_batch_checksum: batch dims do not match shape");
  const device::Buffer db = device::upload(batch), df = device::upload(filters);
  device::Buffer out(static_cast<std::size_t>(ls.k * ls.p * ls.q) * 8);
  const abed_layer_shape s = device::c_shape(ls);
  device::check(abed_conv_batch_checksum(db.get<int32_t>(), df.get<int8_t>(), &s, out.get<int64_t>(), nullptr));
  return device::download(out, {1, ls.k, ls.p, ls.q}, ElemKind::I64);
}

inline VerifyOutcome ic_batch_verify(const Tensor4D& convout, const Tensor4D& extra) {
  if (convout.kind() != ElemKind::I32) throw std::invalid_argument("ic_batch_verify: convout must be i32");
  if (extra.kind() != ElemKind::I64) throw std::invalid_argument("ic_batch_verify: extra batch must be i64");
  const Dims4 d = convout.dims();
  if (extra.dims() != Dims4{1, d.d1, d.d2, d.d3})
    throw std::invalid_argument("ic_batch_verify: extra batch dims do not match convout");
  const device::Buffer dc = device::upload(convout), de = device::upload(extra);
  abed_verify_outcome o{};
  device::check(abed_ic_batch_verify(dc.get<int32_t>(), device::c_dims(d), de.get<int64_t>(), &o));
  return detail::from_c(o);
}

// ------------------------------------------------------------------ planner
struct PrecisionPlan {
  int operand_bits = 8;
  int bits_output_fmap = 0, bits_reduced_fc = 0, bits_reduced_fic = 0;
  int bits_filter_checksum = 0, bits_input_checksum = 0;
  ElemKind output_fmap_kind = ElemKind::I32, reduced_fc_kind = ElemKind::I64, reduced_fic_kind = ElemKind::I64;
  ElemKind filter_checksum_kind = ElemKind::I32, input_checksum_kind = ElemKind::I32;
};

inline PrecisionPlan plan_precision(const LayerShape& ls, int operand_bits) {
  const abed_layer_shape s = device::c_shape(ls);
  abed_precision_plan p{};
  device::check(abed_plan_precision(&s, operand_bits, &p));
  auto k = [](int32_t v) { return static_cast<ElemKind>(v); };
  return PrecisionPlan{p.operand_bits, p.bits_output_fmap, p.bits_reduced_fc, p.bits_reduced_fic,
                       p.bits_filter_checksum, p.bits_input_checksum, k(p.output_fmap_kind), k(p.reduced_fc_kind),
                       k(p.reduced_fic_kind), k(p.filter_checksum_kind), k(p.input_checksum_kind)};
}

// ------------------------------------------------------------------ float mode
inline VerifyOutcome float_verify(double lhs, double rhs, double tau) {
  abed_verify_outcome o{};
  device::check(abed_float_verify(lhs, rhs, tau, &o));
  return detail::from_c(o);
}

inline std::vector<double> filter_checksum_f64(const Tensor4D& filters) {
  if (filters.kind() != ElemKind::F32) throw std::invalid_argument("filter_checksum_f64: expected f32 filters");
  const Dims4 d = filters.dims();
  const std::size_t n = static_cast<std::size_t>(d.d1 * d.d2 * d.d3);
  const device::Buffer df = device::upload(filters);
  device::Buffer out(n * 8);
  device::check(abed_filter_checksum_f64(df.get<float>(), device::c_dims(d), out.get<double>(), nullptr));
  std::vector<double> h(n);
  device::download(out, h.data(), n * 8);
  return h;
}

inline std::vector<double> input_checksum_f64(const Tensor4D& input, const LayerShape& ls) {
  if (input.kind() != ElemKind::F32 || input.dims() != ls.input_dims())
    throw std::invalid_argument("input_checksum_f64: input does not match shape");
  const std::size_t n = static_cast<std::size_t>(ls.crs());
  const device::Buffer dx = device::upload(input);
  device::Buffer out(n * 8);
  const abed_layer_shape s = device::c_shape(ls);
  device::check(abed_input_checksum_f64(dx.get<float>(), &s, out.get<double>(), nullptr));
  std::vector<double> h(n);
  device::download(out, h.data(), n * 8);
  return h;
}

inline double reduce_all_f64(const Tensor4D& convout) {
  const device::Buffer dc = device::upload(convout);
  double r = 0;
  device::check(abed_reduce_all_f64(dc.get<float>(), convout.count(), &r));
  return r;
}

inline double fic_dot_f64(const std::vector<double>& a, const std::vector<double>& b) {
  if (a.size() != b.size()) throw std::invalid_argument("fic_dot_f64: size mismatch");
  const device::Buffer da = device::upload(a.data(), a.size() * 8), db = device::upload(b.data(), b.size() * 8);
  double r = 0;
  device::check(abed_fic_dot_f64(da.get<double>(), db.get<double>(), static_cast<int64_t>(a.size()), &r));
  return r;
}

inline VerifyOutcome fic_verify_f32(const Tensor4D& convout, double expected, double tau) {
  const device::Buffer dc = device::upload(convout);
  abed_verify_outcome o{};
  device::check(abed_fic_verify_f32(dc.get<float>(), convout.count(), expected, tau, &o));
  return detail::from_c(o);
}

inline VerifyOutcome fc_verify_f32(const Tensor4D& convout, const Tensor4D& extra, double tau) {
  if (convout.kind() != ElemKind::F32 || extra.kind() != ElemKind::F32)
    throw std::invalid_argument("fc_verify_f32: expected f32 tensors");
  const Dims4 d = convout.dims();
  if (extra.dims() != Dims4{d.d0, 1, d.d2, d.d3}) throw std::invalid_argument("fc_verify_f32: extra fmap dims do not match convout");
  const device::Buffer dc = device::upload(convout), de = device::upload(extra);
  abed_verify_outcome o{};
  device::check(abed_fc_verify_f32(dc.get<float>(), device::c_dims(d), de.get<float>(), tau, &o));
  return detail::from_c(o);
}

inline VerifyOutcome ic_verify_k_f32(const Tensor4D& convout, const Tensor4D& filters, const std::vector<double>& ic,
                                     double tau) {
  if (convout.kind() != ElemKind::F32 || filters.kind() != ElemKind::F32)
    throw std::invalid_argument("ic_verify_k_f32: expected f32 tensors");
  const Dims4 fd = filters.dims();
  if (static_cast<std::int64_t>(ic.size()) != fd.d1 * fd.d2 * fd.d3)
    throw std::invalid_argument("ic_verify_k_f32: checksum size does not match filters");
  const device::Buffer dc = device::upload(convout), df = device::upload(filters), di = device::upload(ic.data(), ic.size() * 8);
  abed_verify_outcome o{};
  device::check(abed_ic_verify_k_f32(dc.get<float>(), device::c_dims(convout.dims()), df.get<float>(), device::c_dims(fd),
                                     di.get<double>(), tau, &o));
  return detail::from_c(o);
}

// ------------------------------------------------------------------ fused conv + epilog
struct FusedTaps {
  bool output_checksum = false;
  std::optional<LayerShape> next_layer;
};

struct FusedConvResult {
  Tensor4D output;
  std::optional<std::int64_t> output_checksum;
  std::optional<InputChecksum> next_input_checksum;
};

/// One launch of the fused tcgen05 kernel (conv -> output-checksum reduction ->
/// bias/ReLU/requant); the AF tap then computes the next layer's input checksum.
inline FusedConvResult fused_conv_epilog(const Tensor4D& input, const Tensor4D& filters, const LayerShape& ls,
                                         const EpilogParams& params, const FusedTaps& taps = {}) {
  detail::check_conv_args(input, filters, ls, ElemKind::I8, ElemKind::I8);
  if (static_cast<std::int64_t>(params.bias.size()) != ls.k)
    throw std::invalid_argument("epilog: bias length must equal the channel count");
  const detail::DeviceEpilog ep(params);
  const device::Buffer dx = device::upload(input), df = device::upload(filters);
  const std::size_t out_bytes = static_cast<std::size_t>(ls.nkpq()) * elem_size(params.output_kind);
  device::Buffer out(out_bytes);
  std::int64_t cs = 0;
  std::optional<abed_layer_shape> next;
  if (taps.next_layer) next = device::c_shape(*taps.next_layer);
  device::Buffer nic(next ? static_cast<std::size_t>(taps.next_layer->crs()) * 4 : 16);
  const abed_layer_shape s = device::c_shape(ls);
  device::check(abed_fused_conv_epilog(dx.get<int8_t>(), df.get<int8_t>(), &s, &ep.c, out.get(),
                                       taps.output_checksum ? &cs : nullptr, next ? &*next : nullptr,
                                       next ? nic.get<int32_t>() : nullptr, nullptr));
  FusedConvResult r;
  r.output = device::download(out, ls.output_dims(), params.output_kind);
  if (taps.output_checksum) r.output_checksum = cs;
  if (next) {
    const LayerShape& nl = *taps.next_layer;
    r.next_input_checksum = InputChecksum{device::download(nic, {1, nl.c, nl.r, nl.s}, ElemKind::I32)};
  }
  return r;
}

}  // namespace abed
