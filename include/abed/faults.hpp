// abed/faults.hpp -- drop-in for the reference's faults.hpp (fault injection).
//
// flip_bit / flip_bit_inplace (:53-69) act on host tensors exactly as the
// reference does.  run_trial (:268) and run_campaign (:276) run on the B200:
// golden pass once, then per trial a seeded single-bit flip applied in device
// memory (packed input / packed filters / the ConvOut accumulator inside the
// fused epilogue) followed by the fused conv with the scheme's check and the
// epilog.  Reports are identical to the reference's for the same config
// (tests/test_gpu_parity.py: acceptance campaign counts).
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>

#include "checksum.hpp"
#include "convolution.hpp"
#include "device.hpp"
#include "rng.hpp"
#include "tensor.hpp"

namespace abed {

enum class InjectionTarget { InputFmap, Filter, ConvOut };
inline const char* to_string(InjectionTarget t) {
  constexpr const char* names[] = {"input", "filter", "convout"};
  return names[static_cast<int>(t)];
}

enum class Classification { Detected, SDC, Masked, DetectedBenign };
inline const char* to_string(Classification c) {
  constexpr const char* names[] = {"detected", "sdc", "masked", "detected_benign"};
  return names[static_cast<int>(c)];
}

struct FlipSpec {
  InjectionTarget target = InjectionTarget::ConvOut;
  std::int64_t flat_index = 0;
  int bit = 0;
};

struct TrialOutcome {
  Classification classification = Classification::Masked;
  FlipSpec flipped;
  bool final_output_differs = false;
  VerifyOutcome verify;
};

inline void flip_bit_inplace(Tensor4D& t, std::int64_t flat_index, int bit) {
  if (flat_index < 0 || flat_index >= t.count()) throw std::out_of_range("flip_bit: flat index out of bounds");
  if (bit < 0 || bit >= elem_bits(t.kind())) throw std::out_of_range("flip_bit: bit position out of range for element kind");
  auto* b = reinterpret_cast<std::uint8_t*>(t.raw());
  b[static_cast<std::size_t>(flat_index) * elem_size(t.kind()) + static_cast<std::size_t>(bit / 8)] ^=
      static_cast<std::uint8_t>(1u << (bit % 8));
}

inline Tensor4D flip_bit(const Tensor4D& t, std::int64_t flat_index, int bit) {
  Tensor4D out = t;
  flip_bit_inplace(out, flat_index, bit);
  return out;
}

enum class DataMode { Ones, RandomI8 };
inline const char* to_string(DataMode m) { return m == DataMode::Ones ? "ones" : "random"; }

struct CampaignConfig {
  LayerShape shape;
  Scheme scheme = Scheme::FIC;
  InjectionTarget target = InjectionTarget::ConvOut;
  std::int64_t trials = 1000;
  std::uint64_t root_seed = 1;
  DataMode mode = DataMode::Ones;
  EpilogParams epilog;  // bias resized to K when empty
  int jobs = 0;         // accepted for API parity; the GPU batches trials itself
};

struct CampaignReport {
  Scheme scheme = Scheme::FIC;
  InjectionTarget target = InjectionTarget::ConvOut;
  std::int64_t trials = 0, detected = 0, detected_benign = 0, sdc = 0, masked = 0;
  std::uint64_t seed = 0;
  double detection_rate() const {
    return trials ? static_cast<double>(detected + detected_benign) / static_cast<double>(trials) : 0.0;
  }
  double sdc_rate() const { return trials ? static_cast<double>(sdc) / static_cast<double>(trials) : 0.0; }
  bool operator==(const CampaignReport&) const = default;
};

inline TrialOutcome run_trial(const LayerShape& ls, const Tensor4D& input, const Tensor4D& filters, Scheme scheme,
                              InjectionTarget target, const EpilogParams& params, std::uint64_t seed) {
  detail::check_conv_args(input, filters, ls, ElemKind::I8, ElemKind::I8);
  const device::Buffer dx = device::upload(input), df = device::upload(filters);
  const abed_layer_shape s = device::c_shape(ls);
  abed_trial_outcome o{};
  device::check(abed_run_trial(&s, dx.get<int8_t>(), df.get<int8_t>(), static_cast<int32_t>(scheme),
                               static_cast<int32_t>(target), params.scale, params.bias.empty() ? nullptr : params.bias.data(),
                               static_cast<int64_t>(params.bias.size()),
                               params.activation == Activation::ReLU ? ABED_RELU : ABED_IDENTITY,
                               static_cast<int32_t>(params.output_kind), seed, &o));
  TrialOutcome t;
  t.classification = static_cast<Classification>(o.classification);
  t.flipped = FlipSpec{static_cast<InjectionTarget>(o.target), o.flat_index, o.bit};
  t.final_output_differs = o.final_output_differs != 0;
  t.verify = detail::from_c(o.verify);
  return t;
}

/// Trials [begin, end) of a campaign; per-trial seeds derive_seed(root, t), so any
/// split across GPUs folds to the full report (sum the counts).
inline CampaignReport run_campaign_range(const CampaignConfig& cfg, std::int64_t begin, std::int64_t end) {
  const abed_campaign_config c{device::c_shape(cfg.shape), static_cast<int32_t>(cfg.scheme), static_cast<int32_t>(cfg.target),
                               cfg.trials, cfg.root_seed, static_cast<int32_t>(cfg.mode), cfg.epilog.scale,
                               cfg.epilog.bias.empty() ? nullptr : cfg.epilog.bias.data(),
                               static_cast<int64_t>(cfg.epilog.bias.size()),
                               cfg.epilog.activation == Activation::ReLU ? ABED_RELU : ABED_IDENTITY,
                               static_cast<int32_t>(cfg.epilog.output_kind), cfg.jobs};
  abed_campaign_report r{};
  device::check(abed_run_campaign(&c, begin, end, &r));
  CampaignReport rep;
  rep.scheme = static_cast<Scheme>(r.scheme);
  rep.target = static_cast<InjectionTarget>(r.target);
  rep.trials = r.trials;
  rep.detected = r.detected;
  rep.detected_benign = r.detected_benign;
  rep.sdc = r.sdc;
  rep.masked = r.masked;
  rep.seed = r.seed;
  return rep;
}

inline CampaignReport run_campaign(const CampaignConfig& cfg) {
  if (cfg.trials < 1) throw std::invalid_argument("run_campaign: trials must be >= 1");
  return run_campaign_range(cfg, 0, cfg.trials);
}

}  // namespace abed
