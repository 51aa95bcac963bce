// abed/protected_conv.hpp -- device-resident protected layer (the hot path).
//
// Beyond the reference's value-semantics API (checksum.hpp fused_conv_epilog),
// production users keep activations on the GPU: a ProtectedConv owns the packed
// filters (+ FC checksum-digit rows, the offline filter checksum, SPEC "computed
// once offline") and runs the fused tcgen05 conv + FC/FIC/IC verification +
// bias/ReLU/requant epilog on caller-owned device buffers and a CUDA stream.
#pragma once

#include <array>
#include <cstdint>

#include "checksum.hpp"
#include "device.hpp"

namespace abed {

class ProtectedConv {
 public:
  /// filters_dev: KCRS int8 device pointer; checks: ABED_CHECK_FC | ABED_CHECK_FIC | ABED_CHECK_IC
  ProtectedConv(const LayerShape& ls, const std::int8_t* filters_dev, int checks) : ls_(ls), checks_(checks) {
    const abed_layer_shape s = device::c_shape(ls);
    device::check(abed_conv_plan_create(&s, filters_dev, checks, 0, &plan_));
    device::check(abed_conv_plan_info(plan_, &info_));
    outcomes_ = device::Buffer(3 * sizeof(abed_verify_outcome));
  }
  ~ProtectedConv() { abed_conv_plan_destroy(plan_); }
  ProtectedConv(const ProtectedConv&) = delete;
  ProtectedConv& operator=(const ProtectedConv&) = delete;

  std::int64_t packed_input_bytes() const { return info_.packed_input_bytes; }
  const abed_plan_info& info() const { return info_; }
  abed_conv_plan* handle() const { return plan_; }

  /// NCHW int8 device tensor -> packed strip-plane layout (device).
  void pack(const std::int8_t* input_dev, std::int8_t* packed_dev, void* stream = nullptr) const {
    device::check(abed_pack_input(plan_, input_dev, packed_dev, stream));
  }
  /// Fused conv + checks + epilog.  out_mode: ABED_OUT_*; next: consumer layer for ABED_OUT_I8_PACKED.
  void run(const std::int8_t* packed_dev, const abed_epilog_params& ep, int out_mode, void* out_dev,
           const ProtectedConv* next = nullptr, void* stream = nullptr) {
    device::check(abed_conv_plan_run(plan_, packed_dev, &ep, out_mode, out_dev, next ? next->plan_ : nullptr, -1, 0, stream));
    device::check(abed_conv_plan_finalize(plan_, outcomes_.get<abed_verify_outcome>(), stream));
  }
  /// {FC, FIC, IC} outcomes of the last run (synchronous read-back).
  std::array<VerifyOutcome, 3> verdicts() const {
    std::array<abed_verify_outcome, 3> h{};
    device::download(outcomes_, h.data(), sizeof(h));
    return {detail::from_c(h[0]), detail::from_c(h[1]), detail::from_c(h[2])};
  }

 private:
  LayerShape ls_;
  int checks_;
  abed_conv_plan* plan_ = nullptr;
  abed_plan_info info_{};
  device::Buffer outcomes_;
};

}  // namespace abed
