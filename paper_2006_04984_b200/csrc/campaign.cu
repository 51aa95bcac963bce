// C ABI: tensor-core batch checksum, fused conv+epilog with taps, and the GPU
// fault-injection trial / campaign driver.
//
//  * abed_conv_batch_checksum (checksum.hpp:367-396): the ICBatch checksum image
//    sum_n x (|.| <= 128 N) is split into four balanced int8 digit images and
//    convolved on the tcgen05 path as an extra batch; the digit results are
//    recombined in int64 (linearity keeps it exact).
//  * abed_fused_conv_epilog (checksum.hpp:616-631): the protected plan with the
//    FIC reduction supplies the pre-epilog output checksum tap.
//  * abed_run_trial / abed_run_campaign (faults.hpp:197-333): golden run once,
//    then per trial one seeded single-bit flip applied IN DEVICE MEMORY (packed
//    input plane, packed filter block + the KCRS copy the IC verify reads, or the
//    ConvOut accumulator inside the fused epilogue), the fused conv with the
//    scheme's check, the epilog, and an on-device output compare.  Checksums
//    come from the pristine data (faults.hpp:111-115).  Trial seeds are
//    derive_seed(root, t), so reports are identical for any trial sharding.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "abed_internal.h"

using namespace abed_host;
using abed_dev::ActGeom;

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
struct HostRng {  // rng.hpp:11-37
  uint64_t s;
  uint64_t next() { return mix64(s += kGolden); }
  uint64_t below(uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
      const uint64_t r = next();
      if (r >= threshold) return r % bound;
    }
  }
};
uint64_t derive(uint64_t root, uint64_t i) { return HostRng{root ^ (0xA02E9D4BD1C96D4FULL + i * kGolden)}.next(); }

__global__ void digits_kernel(const int32_t* __restrict__ b, int64_t n, int8_t* __restrict__ d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = b[i];
    for (int j = 0; j < 4; ++j) {  // v = sum_j d_j 256^j, d_j in [-128, 127]
      const int32_t dj = ((v + 128) & 0xFF) - 128;
      d[j * n + i] = (int8_t)dj;
      v = (v - dj) / 256;
    }
  }
}
__global__ void recombine_digits_kernel(const int32_t* __restrict__ e, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)e[i] + (int64_t)e[n + i] * 256 + (int64_t)e[2 * n + i] * 65536 + (int64_t)e[3 * n + i] * 16777216;
}
__global__ void xor_byte_kernel(int8_t* a, int64_t ia, int8_t* b, int64_t ib, uint8_t mask) {
  if (a) a[ia] ^= (int8_t)mask;
  if (b) b[ib] ^= (int8_t)mask;
}
__global__ void differ_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b, int64_t n16, int* flag) {
  int d = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 x = a[i], y = b[i];
    d |= (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
  }
  if (__any_sync(0xffffffffu, d) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <typename T>
struct Dev {
  T* p = nullptr;
  explicit Dev(size_t n) { cuda_check(cudaMalloc(&p, (n ? n : 1) * sizeof(T)), "cudaMalloc"); }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

struct PlanGuard {
  abed_conv_plan* p;
  ~PlanGuard() { abed_conv_plan_destroy(p); }
};

// run the tcgen05 conv over NCHW device tensors, int32 NCHW out
void tc_conv_nchw(const abed_layer_shape& s, const int8_t* x, const int8_t* f, int32_t* out, cudaStream_t st) {
  PlanGuard pl{plan_create(s, f, 0, 0)};
  Dev<int8_t> packed((size_t)geom_packed_bytes(pl.p->g));
  abed_pack_input(pl.p, x, packed.p, st);
  plan_run(pl.p, packed.p, nullptr, ABED_OUT_I32_NCHW, out, nullptr, -1, 0, st);
  cuda_check(cudaStreamSynchronize(st), "tc_conv sync");
}

int scheme_checks(int scheme) {
  switch (scheme) {
    case ABED_FC: return ABED_CHECK_FC;
    case ABED_IC: return ABED_CHECK_IC;
    case ABED_FIC: return ABED_CHECK_FIC;
    default: throw_invalid("run_trial: batch-checksum IC is not an injection scheme");
  }
}
int scheme_slot(int scheme) { return scheme == ABED_FC ? 0 : scheme == ABED_FIC ? 1 : 2; }

// faults.hpp:116-130 TrialContext, device resident
struct GpuTrialCtx {
  abed_layer_shape s{};
  int scheme = 0, out_kind = ABED_I8;
  abed_conv_plan* plan = nullptr;
  int8_t* packed = nullptr;
  void* golden = nullptr;
  void* trial_out = nullptr;
  float* bias = nullptr;
  abed_epilog_params ep{};
  int64_t out_bytes = 0;
  ~GpuTrialCtx() {
    abed_conv_plan_destroy(plan);
    cudaFree(packed); cudaFree(golden); cudaFree(trial_out); cudaFree(bias);
  }
};

void ctx_make(GpuTrialCtx& c, const abed_layer_shape& s, const int8_t* x, const int8_t* f, int scheme, float scale,
              const float* bias_host, int64_t bias_len, int act, int kind, cudaStream_t st) {
  validate_shape(s);
  c.s = s;
  c.scheme = scheme;
  const int checks = scheme_checks(scheme);
  if (kind != ABED_I8 && kind != ABED_F32) throw_invalid("epilog: output kind must be i8 or f32");
  if (!std::isfinite(scale)) throw_invalid("epilog: non-finite scale");
  std::vector<float> hb((size_t)s.k, 0.0f);  // faults.hpp:167-168: empty bias -> zeros
  if (bias_host && bias_len > 0) {
    if (bias_len != s.k) throw_invalid("epilog: bias length must equal the channel count");
    for (int64_t i = 0; i < s.k; ++i) {
      if (!std::isfinite(bias_host[i])) throw_invalid("epilog: non-finite bias");
      hb[(size_t)i] = bias_host[i];
    }
  }
  c.out_kind = kind;
  cuda_check(cudaMalloc(&c.bias, (size_t)s.k * 4), "cudaMalloc(bias)");
  cuda_check(cudaMemcpy(c.bias, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice), "bias h2d");
  c.ep = abed_epilog_params{scale, c.bias, s.k, act, kind};
  c.plan = plan_create(s, f, checks, 0);
  cuda_check(cudaMalloc(&c.packed, (size_t)geom_packed_bytes(c.plan->g)), "cudaMalloc(packed)");
  abed_pack_input(c.plan, x, c.packed, st);
  const int64_t nkpq = s.n * s.k * s.p * s.q;
  c.out_bytes = (nkpq * (kind == ABED_F32 ? 4 : 1) + 15) / 16 * 16;
  cuda_check(cudaMalloc(&c.golden, (size_t)c.out_bytes), "cudaMalloc(golden)");
  cuda_check(cudaMalloc(&c.trial_out, (size_t)c.out_bytes), "cudaMalloc(trial)");
  cuda_check(cudaMemsetAsync(c.golden, 0, (size_t)c.out_bytes, st), "memset");
  cuda_check(cudaMemsetAsync(c.trial_out, 0, (size_t)c.out_bytes, st), "memset");
  // golden run: checksums from the pristine input, golden output
  c.plan->reuse_input_checksum = 0;
  c.plan->pdl = 0;  // trials patch filter storage right before each run
  plan_run(c.plan, c.packed, &c.ep, kind == ABED_F32 ? ABED_OUT_F32_NCHW : ABED_OUT_I8_NCHW, c.golden, nullptr, -1, 0, st);
  {
    // the verdict reduction of the golden run keeps its FIC rhs (pristine input
    // checksum) for the trials, which reuse it (faults.hpp:111-115)
    Dev<abed_verify_outcome> scratch(3);
    plan_finalize(c.plan, scratch.p, st);
    cuda_check(cudaStreamSynchronize(st), "golden verdict");
  }
  c.plan->reuse_input_checksum = 1;
  cuda_check(cudaStreamSynchronize(st), "golden run");
}

// one trial, asynchronous; outcome -> out3 (3 slots), differs -> flag
void trial_enqueue(GpuTrialCtx& c, int target, int64_t flat, int bit, abed_verify_outcome* out3, int* flag,
                   cudaStream_t st) {
  const abed_layer_shape& s = c.s;
  const ActGeom& g = c.plan->g;
  const abed_dev::ConvTcParams& p = c.plan->base;
  int8_t* a = nullptr;
  int8_t* b = nullptr;
  int64_t ia = 0, ib = 0;
  int64_t fault_key = -1;
  const uint8_t mask = (uint8_t)(1u << (bit % 8));
  if (target == ABED_TARGET_INPUT) {
    const int64_t w = flat % s.w, h = (flat / s.w) % s.h, ch = (flat / (s.w * s.h)) % s.c, n = flat / (s.w * s.h * s.c);
    const int64_t hp = h + s.pad_h, wp = w + s.pad_w;
    const int ph_a = (int)(hp % s.stride_h), ph_b = (int)(wp % s.stride_w);
    if (ph_a < g.nph_h && ph_b < g.nph_w) {  // pixels of untouched phases are never read by the conv
      const int64_t t = (n * g.Hl + hp / s.stride_h) * g.Wl + wp / s.stride_w;
      const int64_t plane = (int64_t)(ph_a * g.nph_w + ph_b) * g.c16 + ch / 16;
      a = c.packed;
      ia = (plane * g.plane_len + t) * 16 + ch % 16;
    }
  } else if (target == ABED_TARGET_FILTER) {
    const int64_t ss = flat % s.s, r = (flat / s.s) % s.r, ch = (flat / (s.s * s.r)) % s.c, k = flat / (s.s * s.r * s.c);
    const int64_t nt = k / p.block_n, row = k % p.block_n, grp = ch / 16, ks = grp / p.gps, gl = grp % p.gps;
    const int64_t tap = r * s.s + ss;
    a = c.plan->d_wpk;
    ia = ((((nt * p.k_stages + ks) * p.ntaps + tap) * p.gps + gl) * p.block_n_tot + row) * 16 + ch % 16;
    b = c.plan->d_filters;  // the IC verify re-reads filter storage (faults.hpp:242-245)
    ib = flat;
  } else {
    fault_key = flat;
  }
  if (a || b) xor_byte_kernel<<<1, 1, 0, st>>>(a, ia, b, ib, mask);
  plan_run(c.plan, c.packed, &c.ep, c.out_kind == ABED_F32 ? ABED_OUT_F32_NCHW : ABED_OUT_I8_NCHW, c.trial_out, nullptr,
           fault_key, bit, st);
  plan_finalize(c.plan, out3, st);
  differ_kernel<<<grid_for(c.out_bytes / 16, 256), 256, 0, st>>>(static_cast<const uint4*>(c.trial_out),
                                                                 static_cast<const uint4*>(c.golden), c.out_bytes / 16, flag);
  if (a || b) xor_byte_kernel<<<1, 1, 0, st>>>(a, ia, b, ib, mask);  // restore pristine data
  cuda_check(cudaGetLastError(), "trial");
}

int classify(int verify_status, int differs) {  // faults.hpp:255-261
  if (verify_status == 0) return differs ? ABED_SDC : ABED_MASKED;
  return differs ? ABED_DETECTED : ABED_DETECTED_BENIGN;
}

void draw(uint64_t seed, const abed_layer_shape& s, int target, int64_t& flat, int& bit) {  // faults.hpp:200-208
  HostRng g{seed};
  const int64_t count = target == ABED_TARGET_INPUT ? s.n * s.c * s.h * s.w
                        : target == ABED_TARGET_FILTER ? s.k * s.c * s.r * s.s
                                                       : s.n * s.k * s.p * s.q;
  flat = (int64_t)g.below((uint64_t)count);
  bit = (int)g.below(target == ABED_TARGET_CONVOUT ? 32u : 8u);
}

}  // namespace

#define GUARD(...)              \
  try {                         \
    require_device();           \
    __VA_ARGS__;                \
    return ABED_OK;             \
  } catch (const AbedError& e) { \
    return set_error(e.code, e.what()); \
  } catch (const std::exception& e) { \
    return set_error(ABED_ERR_RUNTIME, e.what()); \
  }

extern "C" {

int abed_conv_batch_checksum(const int32_t* batch, const int8_t* filters, const abed_layer_shape* shape, int64_t* out,
                             void* stream) {
  GUARD(
      validate_shape(*shape); cudaStream_t st = (cudaStream_t)stream;
      abed_layer_shape four = *shape; four.n = 4;  // four digit images as one batch
      const int64_t chw = shape->c * shape->h * shape->w, kpq = shape->k * shape->p * shape->q;
      Dev<int8_t> dig((size_t)(4 * chw)); Dev<int32_t> e((size_t)(4 * kpq));
      digits_kernel<<<grid_for(chw, 256), 256, 0, st>>>(batch, chw, dig.p);
      tc_conv_nchw(four, dig.p, filters, e.p, st);
      recombine_digits_kernel<<<grid_for(kpq, 256), 256, 0, st>>>(e.p, kpq, out);
      cuda_check(cudaGetLastError(), "conv_batch_checksum"));
}

int abed_fused_conv_epilog(const int8_t* x, const int8_t* f, const abed_layer_shape* s, const abed_epilog_params* ep,
                           void* out, int64_t* out_checksum, const abed_layer_shape* next, int32_t* next_ic, void* stream) {
  GUARD(
      validate_shape(*s); cudaStream_t st = (cudaStream_t)stream;
      if (s->c * s->r * s->s > 65536) throw_invalid("conv_direct: CRS > 65536 exceeds the int32 accumulator plan");
      if (ep->bias_len != s->k) throw_invalid("epilog: bias length must equal the channel count");
      if (!std::isfinite(ep->scale)) throw_invalid("epilog: non-finite scale");
      {
        std::vector<float> hb((size_t)s->k);
        cuda_check(cudaMemcpy(hb.data(), ep->bias, hb.size() * 4, cudaMemcpyDeviceToHost), "bias d2h");
        for (float v : hb) if (!std::isfinite(v)) throw_invalid("epilog: non-finite bias");
      }
      if (ep->output_kind != ABED_I8 && ep->output_kind != ABED_F32) throw_invalid("epilog: output kind must be i8 or f32");
      PlanGuard pl{plan_create(*s, f, out_checksum ? ABED_CHECK_FIC : 0, 0)};
      pl.p->reuse_input_checksum = 1;  // only the output reduction is needed for the tap
      Dev<int8_t> packed((size_t)geom_packed_bytes(pl.p->g));
      abed_pack_input(pl.p, x, packed.p, st);
      plan_run(pl.p, packed.p, ep, ep->output_kind == ABED_F32 ? ABED_OUT_F32_NCHW : ABED_OUT_I8_NCHW, out, nullptr, -1, 0, st);
      if (out_checksum) {
        Dev<abed_verify_outcome> oc(3);
        cuda_check(cudaMemsetAsync(pl.p->d_acc, 0, 8, st), "memset");
        plan_finalize(pl.p, oc.p, st);
        abed_verify_outcome h;
        cuda_check(cudaMemcpyAsync(&h, oc.p + 1, sizeof(h), cudaMemcpyDeviceToHost, st), "d2h");
        cuda_check(cudaStreamSynchronize(st), "sync");
        *out_checksum = h.lhs;
      }
      if (next) {  // checksum.hpp:623-629 AF tap
        if (ep->output_kind != ABED_I8) throw_invalid("fused_conv_epilog: next-layer checksum tap needs an i8 epilog");
        if (next->n != s->n || next->c != s->k || next->h != s->p || next->w != s->q)
          throw_invalid("fused_conv_epilog: next-layer shape does not match the output");
        dev_gen_input_checksum(static_cast<const int8_t*>(out), *next, next_ic, st);
      }
      cuda_check(cudaStreamSynchronize(st), "fused sync"));
}

int abed_run_trial(const abed_layer_shape* s, const int8_t* x, const int8_t* f, int32_t scheme, int32_t target,
                   float scale, const float* bias_host, int64_t bias_len, int32_t act, int32_t kind, uint64_t seed,
                   abed_trial_outcome* out) {
  GUARD(
      cudaStream_t st = nullptr; GpuTrialCtx c;
      ctx_make(c, *s, x, f, scheme, scale, bias_host, bias_len, act, kind, st);
      int64_t flat; int bit; draw(seed, *s, target, flat, bit);
      Dev<abed_verify_outcome> oc(3); Dev<int> flag(1);
      cuda_check(cudaMemset(flag.p, 0, 4), "memset");
      trial_enqueue(c, target, flat, bit, oc.p, flag.p, st);
      abed_verify_outcome h[3]; int differs = 0;
      cuda_check(cudaMemcpy(h, oc.p, sizeof(h), cudaMemcpyDeviceToHost), "d2h");
      cuda_check(cudaMemcpy(&differs, flag.p, 4, cudaMemcpyDeviceToHost), "d2h");
      std::memset(out, 0, sizeof(*out));
      out->target = target; out->flat_index = flat; out->bit = bit; out->final_output_differs = differs;
      out->verify = h[scheme_slot(scheme)];
      out->classification = classify(out->verify.status, differs));
}

int abed_run_campaign(const abed_campaign_config* cfg, int64_t t_begin, int64_t t_end, abed_campaign_report* rep) {
  GUARD(
      if (cfg->trials < 1) throw_invalid("run_campaign: trials must be >= 1");
      const abed_layer_shape& s = cfg->shape; validate_shape(s);
      cudaStream_t st = nullptr;
      const int64_t nchw = s.n * s.c * s.h * s.w, kcrs = s.k * s.c * s.r * s.s;
      Dev<int8_t> x((size_t)nchw), f((size_t)kcrs);
      if (cfg->mode == ABED_DATA_ONES) {
        cuda_check(cudaMemset(x.p, 1, (size_t)nchw), "memset"); cuda_check(cudaMemset(f.p, 1, (size_t)kcrs), "memset");
      } else {  // faults.hpp:284-288: one stream, input then filters
        const uint64_t seed = derive(cfg->root_seed, 0x0DA7Au);
        abed_fill_random_i8(x.p, nchw, seed, 0, st);
        abed_fill_random_i8(f.p, kcrs, seed, (uint64_t)nchw, st);
      }
      GpuTrialCtx c;
      ctx_make(c, s, x.p, f.p, cfg->scheme, cfg->scale, cfg->bias_host, cfg->bias_len, cfg->activation, cfg->output_kind, st);
      if (t_begin < 0) t_begin = 0;
      if (t_end > cfg->trials) t_end = cfg->trials;
      const int64_t nt = t_end > t_begin ? t_end - t_begin : 0;
      Dev<abed_verify_outcome> oc((size_t)(3 * nt)); Dev<int> flags((size_t)nt);
      cuda_check(cudaMemset(flags.p, 0, (size_t)(nt ? nt : 1) * 4), "memset");
      for (int64_t t = 0; t < nt; ++t) {
        int64_t flat; int bit; draw(derive(cfg->root_seed, (uint64_t)(t_begin + t)), s, cfg->target, flat, bit);
        trial_enqueue(c, cfg->target, flat, bit, oc.p + 3 * t, flags.p + t, st);
      }
      std::vector<abed_verify_outcome> h((size_t)(3 * nt)); std::vector<int> hf((size_t)nt);
      if (nt) {
        cuda_check(cudaMemcpy(h.data(), oc.p, h.size() * sizeof(abed_verify_outcome), cudaMemcpyDeviceToHost), "d2h");
        cuda_check(cudaMemcpy(hf.data(), flags.p, hf.size() * 4, cudaMemcpyDeviceToHost), "d2h");
      }
      std::memset(rep, 0, sizeof(*rep));
      rep->scheme = cfg->scheme; rep->target = cfg->target; rep->seed = cfg->root_seed; rep->trials = nt;
      const int slot = scheme_slot(cfg->scheme);
      for (int64_t t = 0; t < nt; ++t) {  // fold in trial order (faults.hpp:319-331)
        switch (classify(h[(size_t)(3 * t + slot)].status, hf[(size_t)t])) {
          case ABED_DETECTED: ++rep->detected; break;
          case ABED_DETECTED_BENIGN: ++rep->detected_benign; break;
          case ABED_SDC: ++rep->sdc; break;
          default: ++rep->masked; break;
        }
      });
}

}  // extern "C"
